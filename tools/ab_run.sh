set -u
mkdir -p gpurun_out
for v in 12 10 12 10; do
  MPL_LIN_GEN_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_l$v.json 2>> gpurun_out/ab_l.err
done
echo done
