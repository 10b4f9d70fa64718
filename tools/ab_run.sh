# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hvp_variants.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in 0 1; do
  timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 >> gpurun_out/ab_prof.txt 2>&1
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab.json 2>> gpurun_out/ab.err
done
echo done
