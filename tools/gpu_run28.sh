set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_explicit.py tests/test_gpu_slabs.py tests/test_gpu_edge.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in rq rp10 rq rp10; do
  echo "== $v" >> gpurun_out/hvp_ab.log
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 >> gpurun_out/hvp_ab.log 2>&1
done
echo done
