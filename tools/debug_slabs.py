"""Step-by-step slab-rank run (cfg1, 2 loopback ranks) with progress prints; for debugging on the box."""
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


def log(r, *a):
    print(f"[rank {r}]", *a, flush=True)


def fn(r):
    ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
    log(r, "created, particles", ctx.num_particles())
    c = ctx.resample(sc.dt)
    log(r, "resampled", c)
    ijk, m, vn, fr = ctx.get_nodes()
    log(r, "nodes", len(m), "owned", int(ctx.get_node_owner().sum()))
    v = ctx.get_velocity()
    g, phi = ctx.gradient(v)
    log(r, "gradient phi", phi)
    ctx.linearize(v)
    h = ctx.hvp(v)
    log(r, "hvp", float(np.abs(h).sum()))
    st = ctx.newton_step(sc.solver)
    log(r, "newton", st["newton_iters"], st["cg_iters"])
    ctx.transfer_to_particles(sc.dt)
    log(r, "g2p done; num_particles", ctx.num_particles())
    ids = ctx.get_particle_ids()
    log(r, "ids", len(ids), ids[:3])
    x, vv, F, G = ctx.get_particles()
    log(r, "particles", x.shape)
    for k in range(3):
        st = ctx.step(sc.dt, sc.solver)
        log(r, "step", k, st["newton_iters"], st["cg_iters"], ctx.num_particles())
    ctx.close()
    return True


with cf.ThreadPoolExecutor(R) as ex:
    print([f.result() for f in [ex.submit(fn, r) for r in range(R)]])
