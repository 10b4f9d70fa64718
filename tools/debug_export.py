"""Slab-rank export checks: after a step, export from the main thread one rank at a time, then
concurrently (debugging aid)."""
import concurrent.futures as cf
import faulthandler
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.enable()
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402

sc = scenes.cfg1(prestrain=True)
cuts = np.array([0, 2, 4], np.int32)
R = 2
grp = mpl.Group(R)


def fn(r):
    ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
    try:
        ctx.step(sc.dt, sc.solver)
    except Exception as e:
        print(f"[rank {r}] FAILED: {e}", flush=True)
        raise
    print(f"[rank {r}] stepped, owned {ctx.num_particles()}", flush=True)
    return ctx


with cf.ThreadPoolExecutor(R) as ex:
    ctxs = [f.result() for f in [ex.submit(fn, r) for r in range(R)]]
for r, ctx in enumerate(ctxs):
    print(f"[main] rank {r} num_particles", ctx.num_particles(), flush=True)
    try:
        ids = ctx.get_particle_ids()
        print(f"[main] rank {r} ids ok", len(ids), ids[:4], flush=True)
    except mpl.MplError as e:
        print(f"[main] rank {r} error: {e}", flush=True)
    x, v, F, G = ctx.get_particles()
    print(f"[main] rank {r} particles ok", x.shape, flush=True)
    b = ctx.get_particle_cells()
    print(f"[main] rank {r} cells ok", b.shape, flush=True)
with cf.ThreadPoolExecutor(R) as ex:
    res = [f.result() for f in [ex.submit(lambda c: len(c.get_particle_ids()), c) for c in ctxs]]
print("[main] concurrent ids ok", res, flush=True)
for c in ctxs:
    c.close()
