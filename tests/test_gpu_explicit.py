"""GPU parity of the explicit integration path (Eq. explicitforce P:117-121,
Alg. 3 "Explicit" lines 1-3):  f_i = -sum_c sum_k V_ck tau_ck grad w_ic,  v^{n+1} = v^n + dt (g + f/m)
on free nodes (Dirichlet nodes prescribed), then Load (Alg. 4).

The oracle side composes oracle.explicit_force (pinned in test_oracle_solver.py against the implicit
gradient at S = stretch(tau), and the O(dt^2) stiff limit) with oracle.prepare's v-hat and
Dirichlet sets and oracle.g2p.  Slab ranks (loopback group, one GPU) must reproduce it on owned nodes."""
import concurrent.futures as cf
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2602_07853_b200 import mpl, scenes

from ._parity import TOL, node_ids, rel_l2
from .test_gpu_parity import small_cfg2, two_material

pytestmark = pytest.mark.gpu


def explicit_oracle(sc):
    grid = oracle.Grid(sc.n, sc.dx, sc.origin)
    un, S, prob, v0 = oracle.prepare(sc, grid)
    f = oracle.explicit_force(grid, len(sc.materials), un.m_c, un.V_ck, un.tau_ck)
    act = un.m_i > 0
    free = act & (prob.freed != 0)
    v1 = v0.copy()
    v1[free] = prob.vhat[free] + sc.dt * f[free] / un.m_i[free][:, None]
    parts = oracle.g2p(grid, sc.dt, un.m_c, v1, sc.x, sc.v, sc.F, sc.G, mat=sc.mat, materials=sc.materials)
    return grid, un, f, v1, parts


def _prestrained(sc):
    """Pre-strained F (non-zero tau) and a sticky floor through the block's two lowest node layers."""
    inf = float("inf")
    floor = scenes.DirichletBox((-inf, -inf, -inf), (inf, 9.0 / 32, inf), (0.0, 0.0, 0.0))
    return dataclasses.replace(sc, F=scenes._prestrain(sc.n_particles, 7).astype(sc.F.dtype), dirichlet=[floor])


SCENES = {
    "cfg1b_fp64": lambda: scenes.cfg1(prestrain=True),
    "cfg1b_fp32": lambda: scenes.cfg1(prestrain=True, precision=32),
    "cfg2s_fp64_dirichlet": lambda: _prestrained(small_cfg2(64)),
    "lawmix_fp64": lambda: two_material(64, (1, 0)),
    "watermix_fp64": lambda: two_material(64, (0, 2)),
    "vmmix_fp64": lambda: two_material(64, (0, 0), (1500.0, 0.0)),  # particle return map in Load
}


@pytest.mark.parametrize("name", list(SCENES))
def test_explicit_step_matches_oracle(name):
    sc = SCENES[name]()
    grid, un, f, v1, parts = explicit_oracle(sc)
    tol = TOL[sc.precision]["grad"]
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    ctx.explicit_velocity()
    ijk, m, vn, fr = ctx.get_nodes()
    nid = node_ids(grid, ijk)
    # dt f / m is the elastic part of the velocity change: compare it where it is resolved
    dv_o = v1[nid] - oracle.prepare(sc, grid)[3][nid]
    v_g = ctx.get_velocity()
    assert rel_l2(v_g, v1[nid]) <= tol
    ctx.close()
    ctx = mpl.from_scene(sc, 0)
    st = ctx.explicit_step(sc.dt)
    assert st["n_cells"] >= (un.m_c > 0).sum()
    xg, vg, Fg, Gg = ctx.get_particles()
    ptol = TOL[sc.precision]["step"]
    for a, b, t in ((xg, parts[0], ptol), (vg, parts[1], ptol), (Fg, parts[2], ptol), (Gg, parts[3], 10 * ptol)):
        assert rel_l2(a, b) <= t
    ctx.close()
    assert np.linalg.norm(dv_o) > 0  # the scene actually exercises the force


def test_explicit_force_nonzero_and_momentum():
    """sum_i grad w_ic = 0 for every cell, so sum_i f_i = 0 (Eq. explicitforce): with no Dirichlet nodes
    the explicit update changes the grid momentum by exactly dt g sum_i m_i (gravity) up to rounding."""
    sc = scenes.cfg1(prestrain=True)
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    _, m, vn, _ = ctx.get_nodes()
    p0 = (m[:, None] * vn).sum(0)  # unloaded momentum sum_i m_i v_i^n
    ctx.explicit_velocity()
    p1 = (m[:, None] * ctx.get_velocity()).sum(0)
    ctx.close()
    grav = np.asarray(sc.gravity) * sc.dt * m.sum()
    scale = np.abs(m[:, None] * vn).sum()
    assert np.allclose(p1 - p0, grav, atol=1e-11 * scale)


@pytest.mark.parametrize("cuts", [[0, 2, 4], [0, 1, 2, 4]])
def test_explicit_slabs_match_oracle(cuts):
    sc = scenes.cfg1(prestrain=True)
    grid, un, f, v1, parts = explicit_oracle(sc)
    cuts = np.asarray(cuts, np.int32)
    R = len(cuts) - 1
    grp = mpl.Group(R)

    def fn(r):
        ctx = mpl.from_scene_rank(sc, r, R, cuts, device=0, group=grp)
        try:
            ctx.resample(sc.dt)
            ctx.explicit_velocity()
            ijk = ctx.get_nodes()[0]
            out = dict(nid=node_ids(grid, ijk), own=ctx.get_node_owner(), v=ctx.get_velocity())
            ctx.transfer_to_particles(sc.dt)
            out["ids"] = ctx.get_particle_ids()
            out["x"], out["pv"], out["F"], out["G"] = ctx.get_particles()
            return out
        finally:
            ctx.close()

    with cf.ThreadPoolExecutor(R) as ex:
        res = [fu.result(timeout=600) for fu in [ex.submit(fn, r) for r in range(R)]]
    grp.close()
    nid = np.concatenate([o["nid"][o["own"] == 1] for o in res])
    v = np.concatenate([o["v"][o["own"] == 1] for o in res])
    assert len(nid) == len(np.unique(nid))
    assert rel_l2(v, v1[nid]) <= TOL[64]["grad"]
    ids = np.concatenate([o["ids"] for o in res])
    order = np.argsort(ids)
    assert np.array_equal(ids[order], np.arange(sc.n_particles))
    for key, ref in (("x", parts[0]), ("pv", parts[1]), ("F", parts[2])):
        assert rel_l2(np.concatenate([o[key] for o in res])[order], ref) <= TOL[64]["step"]


def test_explicit_full_size_windows():
    """The explicit path at the jelly workload's full size (256^3 grid, 1.12 M particles, fp32: the
    configuration of profiles/r01_explicit_jelly.json), pre-strained so that f_i != 0: the oracle recomputes
    v^{n+1} = v-hat + dt f / m on 20^3-cell windows (a cube corner, the cube's interior) and Load of the
    window's particles from the GPU's own v^{n+1}; nodes / particles whose support lies inside a window
    are compared element by element (the windowing of tests/test_gpu_fullsize.py)."""
    import types

    from .test_gpu_fullsize import SIZE, _window

    sc = scenes.by_name("jelly", 32)
    sc = dataclasses.replace(sc, F=scenes._prestrain(sc.n_particles, 7).astype(sc.F.dtype))
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    ijk, m, vn, fr = ctx.get_nodes()
    ctx.explicit_velocity()
    v_g = ctx.get_velocity().astype(np.float64)
    ctx.transfer_to_particles(sc.dt)
    x_g, vp_g, F_g, G_g = ctx.get_particles()
    ctx.close()
    n1, n2 = sc.n[1] + 1, sc.n[2] + 1
    key = (ijk[:, 0].astype(np.int64) * n1 + ijk[:, 1]) * n2 + ijk[:, 2]
    full = types.SimpleNamespace(sc=sc, pos={int(k): i for i, k in enumerate(key)})
    tol, ptol = TOL[32]["grad"], TOL[32]["step"]
    for lo in [(100, 38, 100), (118, 56, 118)]:
        w = _window(full, lo)
        un, prob, grid, gpos = w["un"], w["prob"], w["grid"], w["gpos"]
        act = w["complete"] & (un.m_i > 0)
        assert act.sum() > 100 and np.all(gpos[act] >= 0)
        f = oracle.explicit_force(grid, len(sc.materials), un.m_c, un.V_ck, un.tau_ck)
        free = act & (prob.freed != 0)
        v1 = prob.vhat.copy()
        v1[free] = prob.vhat[free] + sc.dt * f[free] / un.m_i[free][:, None]
        assert np.linalg.norm(sc.dt * f[free] / un.m_i[free][:, None]) > 1e-4 * np.linalg.norm(v1[free])
        assert rel_l2(v_g[gpos[act]], v1[act]) <= tol
        sub = w["sub"]
        lo_ = np.asarray(lo)
        base = np.floor(sub.x.astype(np.float64) / sc.dx - 0.5).astype(np.int64)
        inner = np.all((base >= lo_ + 1) & (base <= lo_ + SIZE - 2), axis=1)
        assert inner.sum() > 100
        vnew = np.zeros((grid.nnodes, 3))
        have = gpos >= 0
        vnew[have] = v_g[gpos[have]]
        x_o, v_o, F_o, G_o = oracle.g2p(grid, sc.dt, un.m_c, vnew, sub.x, sub.v, sub.F, sub.G, clip=True,
                                        mat=sub.mat, materials=sc.materials)
        idx = w["keep"][inner]
        assert rel_l2(x_g[idx], x_o[inner]) <= 1e-2 * ptol
        assert rel_l2(vp_g[idx], v_o[inner]) <= ptol
        assert rel_l2(F_g[idx], F_o[inner]) <= ptol
        scale = max(np.linalg.norm(G_o[inner]), np.linalg.norm(v_o[inner]) / sc.dx)
        assert np.linalg.norm(G_g[idx] - G_o[inner]) <= ptol * scale  # reading r2-b, as at full size
