set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/phase_sweep.py cfg5 > gpurun_out/sweep_cfg5.jsonl 2> gpurun_out/sweep_cfg5.err
timeout 1200 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo done
