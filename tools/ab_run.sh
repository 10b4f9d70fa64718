set -u
mkdir -p gpurun_out
for v in 3 2 3 2; do
  MPL_WZ45_MINB=$v timeout 600 python bench.py --config cfg4_nh --no-cpu-baseline --no-e2e --steps 3 --warmup 3 >> gpurun_out/ab_45_$v.json 2>> gpurun_out/ab_45.err
done
MPL_WZ45_MINB=2 MPL_KC=0 python -m tests._hvp_variant_check cfg2s_fp32 > gpurun_out/ab_45chk.txt 2>&1
echo done
