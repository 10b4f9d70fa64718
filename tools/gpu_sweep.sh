#!/bin/bash
# One gpurun call: bench lines of every BASELINE config (informational; the driver's bench is cfg4).
set -u
mkdir -p gpurun_out/sweep
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e"
$B --config cfg2 --steps 10 --warmup 3 > gpurun_out/sweep/cfg2.json 2>> gpurun_out/sweep/err.log
$B --config cfg2 --precision 64 --steps 10 --warmup 3 > gpurun_out/sweep/cfg2_fp64.json 2>> gpurun_out/sweep/err.log
for p in 1 8 27 64; do
  $B --config cfg3_ppc$p --steps 3 --warmup 3 > gpurun_out/sweep/cfg3_ppc$p.json 2>> gpurun_out/sweep/err.log
done
$B --config cfg4 --precision 64 --steps 3 --warmup 3 > gpurun_out/sweep/cfg4_fp64.json 2>> gpurun_out/sweep/err.log
for c in cfg4_nh cfg4_water cfg4_vm; do
  $B --config $c --steps 3 --warmup 3 > gpurun_out/sweep/$c.json 2>> gpurun_out/sweep/err.log
done
$B --config cfg5B --steps 3 --warmup 1 > gpurun_out/sweep/cfg5B.json 2>> gpurun_out/sweep/err.log
echo done
