set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab.log
for rep in 1 2; do for v in wz wz3; do
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/prof_$v.log 2>&1
  echo "$rep $v $(tail -1 gpurun_out/prof_$v.log)" >> gpurun_out/ab.log
done; done
for v in wz wz3; do MPL_HVP_KERNEL=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -x -q > gpurun_out/pytest_gpu_$v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$v.log; done
echo done
