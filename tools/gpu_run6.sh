set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPL_LOOPBACK_SERIAL=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/debug_slabs.py > gpurun_out/debug_serial.log 2>&1; echo "rc=$?" >> gpurun_out/debug_serial.log
echo done
