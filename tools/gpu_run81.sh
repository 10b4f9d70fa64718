set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for e in 4 2; do for gr in wave res; do
  MPL_PCG_E=$e MPL_PCG_GRID=$gr timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t.json 2>> gpurun_out/bench.err
  echo "E=$e grid=$gr $(python -c "import json;d=json.load(open('gpurun_out/bench_t.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms']['pcg'])")" >> gpurun_out/ab.log
done; done
MPL_PCG_E=2 MPL_PCG_GRID=res timeout 900 python -m tests._hvp_variant_check mix_fp32 >> gpurun_out/ab.log 2>&1
echo done
