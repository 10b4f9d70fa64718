set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in wz wzr wz2 wzr2 rp10; do
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/prof_$v.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in wzr wz2; do MPL_HVP_KERNEL=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k hvp > gpurun_out/pytest_gpu_$v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$v.log; done
echo done
