set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --config cfg4_vm --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_vm.json 2>> gpurun_out/bench.err
timeout 600 python tools/explicit_bench.py > gpurun_out/explicit_jelly.json 2>> gpurun_out/bench.err
echo done
