set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 1 2 4; do
  MPL_P2Q_MINB=$m timeout 600 python tools/phase_sweep.py cfg4 > gpurun_out/sweep_m$m.jsonl 2>> gpurun_out/sweep.err
  echo "minb=$m $(python -c "
import json
for l in open('gpurun_out/sweep_m$m.jsonl'):
    d=json.loads(l); print(d['config'], d['resample_ms'], end='; ')")" >> gpurun_out/ab.log
done
echo done
