# A/B driver for one gpurun call (scratch; edited per experiment)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -x -q -k "bit_exact or index or edge or ragged or empty" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for c in cfg4 cfg3_ppc64; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/res_$c.csv python tools/prof_resample.py $c > gpurun_out/res_$c.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 >> gpurun_out/ab.json 2>> gpurun_out/ab.err
timeout 600 python bench.py --config cfg3_ppc64 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 >> gpurun_out/ab64.json 2>> gpurun_out/ab.err
echo done
