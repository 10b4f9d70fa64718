# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hvp_variants.py tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in 1 2; do
  MPL_VEC_EVENTS=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 >> gpurun_out/ab_ev.json 2>> gpurun_out/ab.err
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab.json 2>> gpurun_out/ab.err
done
echo done
