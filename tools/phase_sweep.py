"""Per-phase timings of the hot path across the BASELINE.json configs (one GPU).

    python tools/phase_sweep.py cfg3_ppc1 cfg3_ppc8 cfg3_ppc27 cfg3_ppc64 cfg4 cfg5

For each config: resample (a0-a4) and G2P (a9) wall time of the synchronous C-ABI calls, one
linearisation (a5), the HVP (a6, mean of 20 back-to-back launches, CUDA events) with its algorithmic
GB/s, and the cost of a fixed amount of Newton-PCG work (1 Newton iteration, 50 PCG iterations, no
line search) so the solver cost can be compared across particle counts (cfg3's PPC sweep: P2Q/G2P
scale with particles, the solve does not).  One JSON line per config.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402


def measure(name: str) -> dict:
    sc = scenes.by_name(name, 32)
    ctx = mpl.from_scene(sc, 0)
    fixed = dict(fixed_newton=1, fixed_cg=[50], fixed_ls=[0])
    ctx.step(sc.dt, sc.solver, **fixed)  # warm-up (allocations, first launches)
    t_res = 1e9
    for _ in range(3):  # best of 3 (each from the same particle state)
        ctx.set_particles(sc.x, sc.v, sc.F, sc.G, sc.vol, sc.mat)
        t0 = time.perf_counter()
        c = ctx.resample(sc.dt)
        t_res = min(t_res, time.perf_counter() - t0)
    v0 = ctx.get_velocity()
    t0 = time.perf_counter()
    ctx.linearize(v0)
    t_lin = time.perf_counter() - t0
    u = np.random.default_rng(4).normal(size=(c.n_nodes, 3)).astype(np.float32)
    hvp_ms = ctx.hvp_bench(u, 20)
    ctx.set_velocity(v0)
    st = ctx.newton_step(sc.solver, **fixed)
    t0 = time.perf_counter()
    ctx.transfer_to_particles(sc.dt)
    t_g2p = time.perf_counter() - t0
    ctx.close()
    nbytes = c.n_cells * 45 * 4 + c.n_nodes * 7 * 4
    return {"config": name, "p2q": os.environ.get("MPL_P2Q", "scatter"), "particles": sc.n_particles, "quadrature_points": c.n_cells, "active_nodes": c.n_nodes,
            "resample_ms": round(t_res * 1e3, 3), "g2p_ms": round(t_g2p * 1e3, 3),
            "linearize_ms": round(t_lin * 1e3, 3), "hvp_us": round(hvp_ms * 1e3, 2),
            "hvp_alg_GBps": round(nbytes / (hvp_ms * 1e-3) / 1e9, 1),
            "hvp_GDOFps": round(3 * c.n_nodes / (hvp_ms * 1e-3) / 1e9, 2),
            "newton1_cg50_ms": round(st["ms_phase"][3] + st["ms_phase"][4] + st["ms_phase"][5], 3),
            "pcg50_ms": round(st["ms_phase"][4], 3)}


if __name__ == "__main__":
    for name in sys.argv[1:] or ["cfg3_ppc1", "cfg3_ppc8", "cfg3_ppc27", "cfg3_ppc64", "cfg4"]:
        print(json.dumps(measure(name)), flush=True)
