set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_slabs.py -x -q > gpurun_out/pytest_slabs.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/pytest_slabs.log
if [ $rc -eq 0 ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
MPL_HVP_KERNEL=pipe2 timeout 300 python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/plain_prof.log 2>&1 && \
MPL_HVP_KERNEL=pipe2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 2 -c 1 -o gpurun_out/hvp_pipe2b -f \
  python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/ncu_full.log 2>&1
fi
echo done
