set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in group warp; do
  MPL_PCG_MAP=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$m.json 2>> gpurun_out/bench.err
  echo "$m $(python -c "import json;d=json.load(open('gpurun_out/bench_$m.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'])")" >> gpurun_out/ab.log
  MPL_PCG_MAP=$m MPL_VEC_EVENTS=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec_$m.json 2>> gpurun_out/bench.err
  echo "$m vec $(python -c "import json;d=json.load(open('gpurun_out/bench_vec_$m.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'])")" >> gpurun_out/ab.log
done
MPL_PCG_MAP=warp timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -x -q > gpurun_out/pytest_gpu_warp.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_warp.log
echo done
