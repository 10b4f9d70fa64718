set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in def pers; do
  MPL_VEC_KERNEL=$v MPL_VEC_EVENTS=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec_$v.json 2>> gpurun_out/bench.err
done
MPL_VEC_KERNEL=pers timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pers.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pers.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_update1 -s 20 -c 1 -o gpurun_out/upd1_full -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo done
