# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
for v in 12 8 12 8; do
  MPL_LIN_GEN_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_lin$v.json 2>> gpurun_out/ab_lin.err
done
MPL_LIN_GEN_MINB=8 python -m tests._hvp_variant_check cfg2s_fp32 > gpurun_out/ab_lincheck.txt 2>&1
echo done
