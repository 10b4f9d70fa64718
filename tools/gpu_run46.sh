set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for pad in 1 0; do
for v in wz wz2 wzs2; do
  MPL_KZ_PAD=$pad MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 > gpurun_out/prof_${v}_$pad.log 2>&1
  echo "$rep pad=$pad $v $(tail -1 gpurun_out/prof_${v}_$pad.log)" >> gpurun_out/ab.log
done; done; done
MPL_KZ_PAD=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu_pad0.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_pad0.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
