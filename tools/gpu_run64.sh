set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 900 python tools/phase_sweep.py cfg3_ppc1 cfg3_ppc8 cfg3_ppc27 cfg3_ppc64 cfg4 cfg5 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
echo done
