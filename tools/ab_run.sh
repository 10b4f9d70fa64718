# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
for v in 0 1; do
  MPL_HVP_EVENTS=0 MPL_PCG_GRAPH=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_ne$v.json 2>> gpurun_out/ab_ne.err
done
echo done
