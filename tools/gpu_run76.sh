set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rs in 0 1; do
  MPL_L2RESET=$rs timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_rs$rs.json 2>> gpurun_out/bench.err
  echo "rs=$rs $(python -c "import json;d=json.load(open('gpurun_out/bench_rs$rs.json'));print(d['ms_per_step'], d['hvp_ms'], d['e2e'], d['phase_ms'])")" >> gpurun_out/ab.log
done
timeout 900 python tools/phase_sweep.py cfg4 cfg5 > gpurun_out/sweep45.jsonl 2> gpurun_out/sweep.err
echo done
