set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_cfg2.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --config cfg2 --precision 64 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_cfg2_fp64.json 2>> gpurun_out/bench.err
timeout 900 python bench.py --precision 64 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_fp64.json 2>> gpurun_out/bench.err
echo done
