set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 1 8 12 16; do
  MPL_LIN_MINB=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t.json 2>> gpurun_out/bench.err
  echo "minb=$m $(python -c "import json;d=json.load(open('gpurun_out/bench_t.json'));print(d['ms_per_step'], d['phase_ms']['linearize'], d['phase_ms']['line_search'])")" >> gpurun_out/ab.log
done
echo done
