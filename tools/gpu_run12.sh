set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in rp10 pipe2 rp; do
  MPL_HVP_KERNEL=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2>> gpurun_out/bench_variants.err; echo "$v rc=$?" >> gpurun_out/bench_variants.err
done
MPL_HVP_KERNEL=rp10 timeout 300 python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/plain_prof.log 2>&1 && \
MPL_HVP_KERNEL=rp10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hvp -s 2 -c 1 -o gpurun_out/hvp_rp10b -f \
  python tools/prof_hvp.py --config cfg4 --reps 3 > gpurun_out/ncu_full.log 2>&1
echo done
