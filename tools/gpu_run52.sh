set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for rep in 1; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_soa.json 2>> gpurun_out/bench.err
  echo "$rep $(python -c "import json;d=json.load(open('gpurun_out/bench_soa.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'], d['cg_iters'])")" >> gpurun_out/ab.log
done
MPL_VEC_EVENTS=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec.json 2>> gpurun_out/bench.err
echo "vec $(python -c "import json;d=json.load(open('gpurun_out/bench_vec.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'])")" >> gpurun_out/ab.log
echo done
