"""Profiling driver: set up a config, linearise at v^0 and run the HVP kernel `reps` times.
Used under ncu (see profiles/README.md); prints the mean HVP time from CUDA events."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--precision", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
sc = scenes.by_name(a.config, a.precision)
ctx = mpl.from_scene(sc)
c = ctx.resample(sc.dt)
v0 = ctx.get_velocity()
ctx.linearize(v0)
u = np.random.default_rng(4).normal(size=(c.n_nodes, 3)).astype(ctx.dtype)
ms = ctx.hvp_bench(u, a.reps)
nbytes = c.n_cells * 45 * (a.precision // 8) + c.n_nodes * 7 * (a.precision // 8)
print(f"{a.config} fp{a.precision}: cells={c.n_cells} nodes={c.n_nodes} hvp={ms*1e3:.1f} us "
      f"alg={nbytes/1e6:.1f} MB -> {nbytes/(ms*1e-3)/1e9:.0f} GB/s")
