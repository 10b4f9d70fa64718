# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hvp_variants.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for v in 4 3 4 3; do
  echo "minb $v" >> gpurun_out/ab_prof.txt
  MPL_KC_MINB=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 30 >> gpurun_out/ab_prof.txt 2>&1
done
for v in 4 3; do
  MPL_KC_MINB=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_$v.json 2>> gpurun_out/ab.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 2 -c 1 -o gpurun_out/hvp_full -f \
  python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/ncu_full.log 2>&1
echo done
