# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
for v in 0 1 0 1; do
  MPL_VEC_EVENTS=1 MPL_PCG_E2=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 >> gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
done
MPL_PCG_E2=1 python -m tests._hvp_variant_check mix_fp32 > gpurun_out/ab_check.txt 2>&1
echo done
