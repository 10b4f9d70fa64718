set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 8 12; do for c in cfg4_nh cfg4_vm cfg4_water; do
timeout 600 env MPL_LIN_GEN_MINB=$m python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_t.json 2>> gpurun_out/bench.err
echo "m=$m $c $(python -c "import json;d=json.load(open('gpurun_out/bench_t.json'));print(d['ms_per_step'], d['phase_ms']['linearize'], d['phase_ms']['line_search'])")" >> gpurun_out/ab.log
done; done
MPL_LIN_GEN_MINB=12 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
