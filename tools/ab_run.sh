# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
for v in p 0 h ph p 0; do
  MPL_L2WIN=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
done
for v in 1 0; do
  MPL_PDL=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_pdl$v.json 2>> gpurun_out/ab.err
done
echo done
