set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hvp_variants.py -q -m gpu > gpurun_out/pytest_var.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_var.log
timeout 900 python bench.py --precision 64 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_fp64.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --config cfg2 --precision 64 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_cfg2_fp64.json 2>> gpurun_out/bench.err
echo done
