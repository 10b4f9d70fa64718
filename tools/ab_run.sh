# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "step" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in 8 6; do
  MPL_C2PT_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_g$v.json 2>> gpurun_out/ab.err
  MPL_C2PT_MINB=$v timeout 600 python bench.py --config cfg3_ppc64 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 >> gpurun_out/ab64_g$v.json 2>> gpurun_out/ab.err
done
echo done
