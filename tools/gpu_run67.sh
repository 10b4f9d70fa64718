set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for u in 1 2 4; do
  MPL_P2Q_UNROLL=$u timeout 600 python tools/phase_sweep.py cfg4 cfg3_ppc8 > gpurun_out/sweep_u$u.jsonl 2>> gpurun_out/sweep.err
  echo "u=$u $(python -c "
import json
for l in open('gpurun_out/sweep_u$u.jsonl'):
    d=json.loads(l); print(d['config'], d['resample_ms'], end='; ')")" >> gpurun_out/ab.log
done
echo done
