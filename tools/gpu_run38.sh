set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
echo done
