set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPL_LIB=dbg CUDA_LAUNCH_BLOCKING=1 timeout 200 python tools/debug_export.py > gpurun_out/debug_export.log 2>&1; echo "rc=$?" >> gpurun_out/debug_export.log
timeout 200 python tools/debug_export.py > gpurun_out/debug_export2.log 2>&1; echo "rc=$?" >> gpurun_out/debug_export2.log
echo done
