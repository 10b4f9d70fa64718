set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPL_VEC_EVENTS=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec.json 2> gpurun_out/bench.err
MPL_HVP_EVENTS=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_noev.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_def.json 2>> gpurun_out/bench.err
echo done
