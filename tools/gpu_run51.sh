set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for pdl in 1 0; do
  MPL_PDL=$pdl timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pdl$pdl.json 2>> gpurun_out/bench.err
  echo "$rep pdl=$pdl $(python -c "import json;d=json.load(open('gpurun_out/bench_pdl$pdl.json'));print(d['ms_per_step'], d['hvp_ms'], d['phase_ms'])")" >> gpurun_out/ab.log
done; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
