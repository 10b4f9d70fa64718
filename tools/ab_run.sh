set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_hvp_variants.py tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab_f.json 2>> gpurun_out/ab_f.err
timeout 600 python bench.py --config cfg4_nh --no-cpu-baseline --no-e2e --steps 3 --warmup 3 >> gpurun_out/ab_fnh.json 2>> gpurun_out/ab_f.err
echo done
