set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPL_LOOPBACK_TIMEOUT=30 MPL_LIB=dbg timeout 150 python tools/debug_export.py > gpurun_out/debug_export.log 2>&1; echo "rc=$?" >> gpurun_out/debug_export.log
MPL_LOOPBACK_TIMEOUT=60 timeout 1200 python -m pytest tests/test_gpu_slabs.py -x -q > gpurun_out/pytest_slabs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slabs.log
echo done
