set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in rq rq8 rp10; do
  MPL_HVP_KERNEL=$v timeout 300 python tools/prof_hvp.py --config cfg4 --reps 20 >> gpurun_out/hvp_ab.log 2>&1
done
for v in rq rp10; do
  MPL_HVP_KERNEL=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2>> gpurun_out/bench.err
done
echo done
