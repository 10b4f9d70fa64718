set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in rp10 pipe2; do
  MPL_HVP_KERNEL=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2>> gpurun_out/bench_variants.err; echo "$v rc=$?" >> gpurun_out/bench_variants.err
done
timeout 1800 python tools/phase_sweep.py cfg2 cfg3_ppc1 cfg3_ppc8 cfg3_ppc27 cfg3_ppc64 cfg4 cfg5 > gpurun_out/phase_sweep.jsonl 2> gpurun_out/phase_sweep.err
echo done
