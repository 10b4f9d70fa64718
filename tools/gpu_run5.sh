set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/debug_slabs.py > gpurun_out/debug_plain.log 2>&1; echo "rc=$?" >> gpurun_out/debug_plain.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/debug_slabs.py > gpurun_out/debug_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/debug_memcheck.log
echo done
