set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/phase_sweep.py cfg4 cfg5 > gpurun_out/sweep45.jsonl 2> gpurun_out/sweep.err
timeout 900 python tools/phase_sweep.py cfg5 > gpurun_out/sweep5.jsonl 2>> gpurun_out/sweep.err
echo done
