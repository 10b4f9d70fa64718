set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in rq rq8 rp10 rp12 pipe2 pipe3 rq rp10; do
  echo "== $v" >> gpurun_out/hvp_ab.log
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 >> gpurun_out/hvp_ab.log 2>&1
done
MPL_HVP_KERNEL=rq timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_rq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rq.log
echo done
