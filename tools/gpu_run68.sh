set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for d in 1 0; do
  MPL_STRETCH_PASS=$d timeout 600 python tools/phase_sweep.py cfg4 cfg3_ppc8 > gpurun_out/sweep_d$d.jsonl 2>> gpurun_out/sweep.err
  echo "d=$d $(python -c "
import json
for l in open('gpurun_out/sweep_d$d.jsonl'):
    d=json.loads(l); print(d['config'], d['resample_ms'], end='; ')")" >> gpurun_out/ab.log
done
MPL_STRETCH_PASS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu_d1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_d1.log
echo done
