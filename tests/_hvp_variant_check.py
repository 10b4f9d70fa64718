"""Subprocess body of tests/test_gpu_hvp_variants.py: with MPL_HVP_KERNEL / MPL_PCG_MAP / MPL_PDL set in
the environment (the library reads them once per process), check one scene's HVP, Jacobi diagonal and
replayed full step against the oracle.  Prints one line 'OK hvp=<rel> step=<rel>' or raises."""
import sys

import numpy as np

from tests._parity import TOL, Pair, cell_ids, rel_l2
from tests.test_gpu_parity import SCENES, _at, _fp32_scene, _probe


def main(name: str) -> None:
    pair = Pair(_fp32_scene(SCENES[name]()))
    sc = pair.scene
    tol = TOL[sc.precision]
    # unload (a2-a4: the P2Q form is one of the options)
    q = pair.ctx.get_quadrature()
    cid = cell_ids(pair.grid, q["ijk"])
    act = pair.un.m_c[cid] > 0
    for nm, got, want in (("m_c", q["m_c"][act], pair.un.m_c[cid][act]), ("v_c", q["v_c"][act], pair.un.v_c[cid][act]),
                          ("G_c", q["G_c"][act], pair.un.G_c[cid][act]), ("m_i", pair.m, pair.un.m_i[pair.nid]),
                          ("v_i", pair.vn, pair.un.v_i[pair.nid])):
        assert rel_l2(got, want) <= tol["unload"], f"{nm} rel l2 {rel_l2(got, want)}"
    for k in range(len(sc.materials)):
        sel = pair.un.V_ck[k][cid] > 0
        assert rel_l2(q["V_ck"][k][act], pair.un.V_ck[k][cid][act]) <= tol["unload"]
        if np.abs(pair.un.tau_ck[k]).max() > 0:
            assert rel_l2(q["tau_ck"][k][sel], pair.un.tau_ck[k][cid][sel]) <= tol["unload"]
        assert rel_l2(q["S_ck"][k][sel], pair.S[k][cid][sel]) <= tol["unload"]
    v, u = _probe(pair)
    po = _at(pair, v)
    pair.ctx.linearize(pair.to_gpu(v))
    h_o = po.hvp(v, u)
    h_g = pair.ctx.hvp(pair.to_gpu(u))
    e_h = rel_l2(h_g, h_o[pair.nid])
    assert e_h <= tol["hvp"], f"hvp rel l2 {e_h}"
    # elastic part: bar tol |el| + 4 eps |m u| (the rounding of the returned Hu; DESIGN.md §9 r2-a)
    m = pair.un.m_i[:, None]
    el_o = (h_o - m * u)[pair.nid]
    d_el = np.linalg.norm(h_g - pair.m[:, None] * pair.to_gpu(u) - el_o)
    eps = 2.0 ** -24 if sc.precision == 32 else 2.0 ** -53
    bar = tol["hvp"] * np.linalg.norm(el_o) + 4 * eps * np.linalg.norm((m * u)[pair.nid])
    e_el = d_el / np.linalg.norm(el_o)
    assert d_el <= bar, f"elastic hvp rel l2 {e_el} (bar {bar / np.linalg.norm(el_o)})"
    e_d = rel_l2(pair.ctx.get_diag(), po.diag(v)[pair.nid])
    assert e_d <= tol["hvp"], f"diag rel l2 {e_d}"
    # one implicit step with the oracle's Newton / PCG / line-search counts replayed
    st_o = pair.prob.newton(pair.v0, sc.solver)[1]
    v_o, _ = pair.prob.newton(pair.v0, sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    pair.ctx.set_velocity(pair.to_gpu(pair.v0))
    st_g = pair.ctx.newton_step(sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    assert st_g["cg_iters"] == st_o["cg_iters"], (st_g["cg_iters"], st_o["cg_iters"])
    e_s = rel_l2(pair.ctx.get_velocity(), v_o[pair.nid])
    assert e_s <= tol["step"], f"step rel l2 {e_s}"
    print(f"OK hvp={e_h:.3e} elastic={e_el:.3e} diag={e_d:.3e} step={e_s:.3e}")


if __name__ == "__main__":
    main(sys.argv[1])
