set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t.json 2>> gpurun_out/bench.err
echo "$(python -c "import json;d=json.load(open('gpurun_out/bench_t.json'));print(d['ms_per_step'], d['hvp_ms'], d['roofline']['frac'], d['phase_ms']['pcg'])")" >> gpurun_out/ab.log
done
echo done
