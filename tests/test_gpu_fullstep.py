"""Full-step parity at BASELINE.json's full sizes (VERDICT r1 "missing #2"): the whole scene through
the C ABI against the fp64 oracle run over the WHOLE grid (OpenMP colour loops, oracle/mpl_oracle.c),
one implicit step (Alg. 1) with the oracle's Newton / PCG / line-search counts replayed
(amb-19), then Load (Alg. 4):
  * cfg2 (64^3, 884,736 particles) in fp64 — bar 1e-8 — and fp32 — bar 1e-4 (north_star full-step bars);
  * cfg3 at PPC 1 (128^3, 1,404,928 particles) in fp32 — bar 1e-4.
Compared: v^{n+1} on every active node, and every particle's x, v, F after Load; G_p (a difference
quotient of v^{n+1}) against the scale max(|G_p|, |v_p| / dx) (DESIGN.md §9 reading r2-b)."""
import numpy as np
import pytest

import oracle
from paper_2602_07853_b200 import mpl, scenes

from ._parity import TOL, node_ids, rel_l2

pytestmark = pytest.mark.gpu

CASES = [("cfg2", 64), ("cfg2", 32), ("cfg3_ppc1", 32)]


@pytest.mark.parametrize("name,precision", CASES, ids=[f"{n}_fp{p}" for n, p in CASES])
def test_full_scene_step_replayed(name, precision):
    sc = scenes.by_name(name, precision)
    tol = TOL[precision]["step"]
    grid = oracle.Grid(sc.n, sc.dx, sc.origin)
    r = oracle.step(sc)  # adaptive oracle step: its counts are replayed on the GPU
    st_o = r.stats
    assert st_o["converged"] == 1
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    st_g = ctx.newton_step(sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    assert st_g["newton_iters"] == st_o["newton_iters"] and st_g["cg_iters"] == st_o["cg_iters"]
    ijk, _, _, _ = ctx.get_nodes()
    nid = node_ids(grid, ijk)
    v_g = ctx.get_velocity()
    assert rel_l2(v_g, r.v_new[nid]) <= tol
    ctx.transfer_to_particles(sc.dt)
    x_g, vp_g, F_g, G_g = ctx.get_particles()
    ctx.close()
    x_o, vp_o, F_o, G_o = r.particles
    assert rel_l2(x_g, x_o) <= tol
    assert rel_l2(vp_g, vp_o) <= tol
    assert rel_l2(F_g, F_o) <= tol
    scale = max(np.linalg.norm(G_o), np.linalg.norm(vp_o) / sc.dx)
    assert np.linalg.norm(G_g - G_o) <= tol * scale
