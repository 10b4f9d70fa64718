set -u
mkdir -p gpurun_out
bash tools/gpu_measure.sh
for c in cfg4_nh cfg4_water cfg4_vm; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err
done
MPL_VEC_EVENTS=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec.json 2>> gpurun_out/bench.err
timeout 600 python tools/explicit_bench.py > gpurun_out/explicit.json 2>> gpurun_out/bench.err
rm -f gpurun_out/sweep.jsonl
for c in cfg3_ppc1 cfg3_ppc8 cfg3_ppc27 cfg3_ppc64 cfg4 cfg5; do
  timeout 900 python tools/phase_sweep.py $c >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err
done
echo done
