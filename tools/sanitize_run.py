"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck): every default kernel of the
hot path on oracle-sized scenes — resample (both P2Q forms via MPL_P2Q), linearise (exact and PSD),
HVP (k_hvp_wz fp32, k_hvp_wh fp64), PCG, line search, G2P.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07853_b200 import mpl, scenes  # noqa: E402


def two_material(precision):
    n = 16
    cells = scenes.cells_box([4, 2, 4], [12, 10, 12])
    x = scenes.stratified(cells, n, 2, seed=0)
    rng = np.random.default_rng(1)
    v = rng.normal(0, 0.3, size=x.shape)
    F = scenes._prestrain(x.shape[0], 3)
    mat = rng.integers(0, 2, size=x.shape[0]).astype(np.int32)
    floor = scenes.DirichletBox((-1e9, -1e9, -1e9), (1e9, 3 / n, 1e9), (0.0, 0.0, 0.0))
    return scenes._assemble("mix", precision, n, 1e-3, [scenes.Material(1e5, 0.3, 1000.0),
                                                        scenes.Material(3e6, 0.45, 2500.0)],
                            x, v, F, np.zeros((x.shape[0], 9)), mat, 8, [floor], scenes.SolverCfg(), 1)


def run(sc, psd=False):
    ctx = mpl.from_scene(sc, 0)
    solver = dataclasses.replace(sc.solver, psd=psd)
    st = ctx.step(sc.dt, solver)
    ctx.set_particles(sc.x, sc.v, sc.F, sc.G, sc.vol, sc.mat)
    ctx.resample(sc.dt)
    v0 = ctx.get_velocity()
    ctx.set_psd_projection(psd)
    ctx.linearize(v0)
    ctx.hvp(np.ones_like(v0))
    ctx.close()
    print(f"{sc.name} fp{sc.precision} psd={psd}: newton {st['newton_iters']} cg {st['cg_iters']} ok", flush=True)


if __name__ == "__main__":
    run(scenes.cfg1(prestrain=True, precision=32))
    run(two_material(32))
    run(two_material(32), psd=True)
    run(two_material(64))
