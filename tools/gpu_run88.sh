set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 0 1; do for c in cfg4 cfg3_ppc64; do
  MPL_P2Q_PERSIST=$m timeout 600 python tools/phase_sweep.py $c > gpurun_out/sweep_t.jsonl 2>> gpurun_out/sweep.err
  echo "pers=$m $(python -c "
import json
for l in open('gpurun_out/sweep_t.jsonl'):
    d=json.loads(l); print(d['config'], d['resample_ms'], end='; ')")" >> gpurun_out/ab.log
done; done
MPL_P2Q_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
