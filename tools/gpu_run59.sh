set -u
mkdir -p gpurun_out
bash tools/gpu_measure.sh
for c in cfg4_nh cfg4_water cfg4_vm; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err
done
MPL_VEC_EVENTS=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec.json 2>> gpurun_out/bench.err
timeout 600 python tools/explicit_bench.py > gpurun_out/explicit.json 2>> gpurun_out/bench.err
echo done
