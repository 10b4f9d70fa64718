set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 1 4; do for c in cfg4 cfg3_ppc64; do
  MPL_C2P_MINB=$m timeout 600 python tools/phase_sweep.py $c > gpurun_out/sweep_t.jsonl 2>> gpurun_out/sweep.err
  echo "m=$m $(python -c "
import json
for l in open('gpurun_out/sweep_t.jsonl'):
    d=json.loads(l); print(d['config'], d['g2p_ms'], end='; ')")" >> gpurun_out/ab.log
done; done
echo done
