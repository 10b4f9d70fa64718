"""The bench's 8-rank slab configuration (cfg4, balanced cuts) run as 8 loopback ranks on one GPU:
two adaptive steps, then the particle state gathered by id against the one-rank run (a scale check of
the multi-GPU path's logic; the NCCL transport replaces the loopback barrier + copy on a real box)."""
import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = 2
sc = scenes.by_name("cfg4", 32)
one = mpl.from_scene(sc, 0)
st1 = [one.step(sc.dt, sc.solver) for _ in range(steps)]
x1, v1, F1, G1 = one.get_particles()
one.close()
cuts = np.asarray(mpl.slab_cuts(sc, R), np.int32)
grp = mpl.Group(R)


def fn(r):
    ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
    try:
        sts = [ctx.step(sc.dt, sc.solver) for _ in range(steps)]
        return sts, ctx.get_particle_ids(), ctx.get_particles()
    finally:
        ctx.close()


t = time.perf_counter()
with cf.ThreadPoolExecutor(R) as ex:
    res = [f.result(timeout=1800) for f in [ex.submit(fn, r) for r in range(R)]]
grp.close()
ids = np.concatenate([r[1] for r in res])
order = np.argsort(ids)
out = {"ranks": R, "cuts": cuts.tolist(), "wall_s": round(time.perf_counter() - t, 1),
       "all_ids": bool(np.array_equal(np.sort(ids), np.arange(sc.n_particles))),
       "cg_iters_1rank": [s["cg_iters"] for s in st1], "cg_iters_rank0": [s["cg_iters"] for s in res[0][0]]}
for k, ref in enumerate((x1, v1, F1, G1)):
    got = np.concatenate([r[2][k] for r in res])[order]
    d = np.linalg.norm((got.astype(np.float64) - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300)
    out["rel_" + "xvFG"[k]] = float(d)
print(json.dumps(out))
