set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lt in 64 128; do
  MPL_LIN_THREADS=$lt timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_lt$lt.json 2>> gpurun_out/bench.err
  echo "lt=$lt $(python -c "import json;d=json.load(open('gpurun_out/bench_lt$lt.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'])")" >> gpurun_out/ab.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
