set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in wh sel; do
  MPL_HVP_KERNEL64=$v timeout 300 python tools/prof_hvp.py --config cfg4 --precision 64 --reps 20 > gpurun_out/prof64_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/prof64_$v.log)" >> gpurun_out/ab.log
done
timeout 900 python bench.py --precision 64 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4_fp64.json 2>> gpurun_out/bench.err
echo done
