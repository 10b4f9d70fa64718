set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in cfg4_nh cfg4_water; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err
done
MPL_VEC_EVENTS=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_vec.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_b1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1100 -c 1400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo done
