set -u
mkdir -p gpurun_out
for v in 3 2 3 2; do
  MPL_KC_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_mb$v.json 2>> gpurun_out/ab_mb.err
done
MPL_KC_MINB=2 python -m tests._hvp_variant_check cfg2s_fp32 > gpurun_out/ab_mbchk.txt 2>&1
MPL_KC_MINB=2 python -m tests._hvp_variant_check cfg1_fp32 >> gpurun_out/ab_mbchk.txt 2>&1
echo done
