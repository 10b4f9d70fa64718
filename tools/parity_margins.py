"""Measured parity errors (relative L2) of every GPU parity scene, next to the bars of tests/_parity.py.

    python tools/parity_margins.py [scene ...]  > gpurun_out/margins.jsonl

For each scene of tests/test_gpu_parity.SCENES: unload (m_c, v_c, G_c, V_ck, tau_ck, S_ck, m_i, v_i),
gradient, HVP, elastic part of the HVP, diagonal, replayed full step (v^{n+1}, x_p, v_p, F_p, G_p).
Used to set / justify the bars; not a test.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tests import test_gpu_parity as T  # noqa: E402
from tests._parity import Pair, cell_ids, rel_l2  # noqa: E402


def rel_sum(got, want, terms):
    """error relative to the L2 norm of |terms| (the magnitude the sum was formed from)"""
    d = np.linalg.norm((np.asarray(got, np.float64) - want).ravel())
    n = np.linalg.norm(np.asarray(terms, np.float64).ravel())
    return float(d / n) if n > 0 else float(d)


def margins(name):
    sc = T._fp32_scene(T.SCENES[name]())
    pr = Pair(sc)
    out = {"scene": name, "precision": sc.precision}
    q = pr.ctx.get_quadrature()
    cid = cell_ids(pr.grid, q["ijk"])
    act = pr.un.m_c[cid] > 0
    out["m_c"] = rel_l2(q["m_c"][act], pr.un.m_c[cid][act])
    out["v_c"] = rel_l2(q["v_c"][act], pr.un.v_c[cid][act])
    out["G_c"] = rel_l2(q["G_c"][act], pr.un.G_c[cid][act])
    for k in range(len(sc.materials)):
        sel = pr.un.V_ck[k][cid] > 0
        out[f"V_c{k}"] = rel_l2(q["V_ck"][k][act], pr.un.V_ck[k][cid][act])
        if np.abs(pr.un.tau_ck[k]).max() > 0:
            out[f"tau_c{k}"] = rel_l2(q["tau_ck"][k][sel], pr.un.tau_ck[k][cid][sel])
        out[f"S_c{k}"] = rel_l2(q["S_ck"][k][sel], pr.S[k][cid][sel])
    out["m_i"] = rel_l2(pr.m, pr.un.m_i[pr.nid])
    out["v_i"] = rel_l2(pr.vn, pr.un.v_i[pr.nid])
    v, u = T._probe(pr)
    po = T._at(pr, v)
    g_o = po.gradient(v)
    g_g, _ = pr.ctx.gradient(pr.to_gpu(v))
    out["grad"] = rel_l2(g_g, g_o[pr.nid])
    pr.ctx.linearize(pr.to_gpu(v))
    h_o = po.hvp(v, u)
    h_g = pr.ctx.hvp(pr.to_gpu(u))
    out["hvp"] = rel_l2(h_g, h_o[pr.nid])
    m = pr.un.m_i[:, None]
    el_o = (h_o - m * u)[pr.nid]
    el_g = h_g - pr.m[:, None] * pr.to_gpu(u)
    out["hvp_elastic"] = rel_l2(el_g, el_o)
    out["elastic_over_mass"] = float(np.linalg.norm(el_o) / np.linalg.norm((m * u)[pr.nid]))
    out["diag"] = rel_l2(pr.ctx.get_diag(), po.diag(v)[pr.nid])
    st_o = pr.prob.newton(pr.v0, sc.solver)[1]
    v_o, _ = pr.prob.newton(pr.v0, sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    pr.ctx.set_velocity(pr.to_gpu(pr.v0))
    pr.ctx.newton_step(sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    out["v_new"] = rel_l2(pr.ctx.get_velocity(), v_o[pr.nid])
    pr.ctx.transfer_to_particles(sc.dt)
    got = pr.ctx.get_particles()
    want = oracle.g2p(pr.grid, sc.dt, pr.un.m_c, v_o, sc.x, sc.v, sc.F, sc.G, mat=sc.mat, materials=sc.materials)
    for nm, a, b in zip(("x_p", "v_p", "F_p", "G_p"), got, want):
        out[nm] = rel_l2(a, b)
    # G_p relative to the nodal velocities it differentiates: G_p = sum v_i (x) grad w, |grad w| = 1/(4 dx)
    out["G_p_vs_v_over_dx"] = rel_sum(got[3], want[3], np.abs(want[1]) / (4 * sc.dx))
    pr.ctx.close()
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or list(T.SCENES)
    for nm in names:
        print(json.dumps(margins(nm)), flush=True)
