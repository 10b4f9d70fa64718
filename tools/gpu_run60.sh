set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cap in 704 0; do
  MPL_P2Q_CAP=$cap timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cap$cap.json 2>> gpurun_out/bench.err
  echo "cap=$cap $(python -c "import json;d=json.load(open('gpurun_out/bench_cap$cap.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'])")" >> gpurun_out/ab.log
done
MPL_P2Q_CAP=0 timeout 600 python tools/phase_sweep.py > gpurun_out/sweep_cap0.jsonl 2>> gpurun_out/bench.err
timeout 600 python tools/phase_sweep.py > gpurun_out/sweep.jsonl 2>> gpurun_out/bench.err
echo done
