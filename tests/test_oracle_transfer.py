"""Oracle pins, part 2: unload (P2C + C2N, C3/C4) and load (G2P, C8).

Conservation laws, affine reproduction, worked examples, the hourglass
null space and the P:1050 reproduction identity — all independent of the oracle code.
"""
import json
import os

import numpy as np
import pytest

from paper_2602_07853_b200 import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def small_scene(seed=0, n=16, ppc_k=2, lo=4, hi=12, prestrain=False, nmat=1):
    cells = scenes.cells_box([lo] * 3, [hi] * 3)
    x = scenes.stratified(cells, n, ppc_k, seed=seed)
    rng = np.random.default_rng(seed + 100)
    v = rng.normal(0, 0.3, size=(x.shape[0], 3))
    G = rng.normal(0, 2.0, size=(x.shape[0], 9))
    F = scenes._prestrain(x.shape[0], seed + 7) if prestrain else np.tile(np.eye(3).ravel(), (x.shape[0], 1))
    vol = np.full(x.shape[0], (1 / n) ** 3 / ppc_k ** 3)
    mat = (rng.integers(0, nmat, size=x.shape[0])).astype(np.int32)
    mats = [scenes.Material(1e4 * (k + 1), 0.3, 1000.0 * (1 + 0.5 * k)) for k in range(nmat)]
    return n, x, v, F, G, vol, mat, mats


def test_unload_conservation(orc):
    """sum m_c = sum m_p; sum (mv)_c = sum m_p v_p (first moment); sum_c V_ck tau_ck =
    sum_{p in k} V_p tau_p (Eq. vtau); then C2N: sum m_i = sum m_p, sum m_i v_i = sum m_p v_p."""
    n, x, v, F, G, vol, mat, mats = small_scene(prestrain=True, nmat=2)
    g = orc.Grid((n,) * 3, 1 / n)
    un = orc.unload(g, mats, x, v, F, G, vol, mat)
    rho = np.array([m.rho for m in mats])[mat]
    mp = rho * vol
    assert un.m_c.sum() == pytest.approx(mp.sum(), rel=1e-13)
    assert np.allclose(un.mv_c.sum(0), (mp[:, None] * v).sum(0), rtol=1e-12, atol=1e-14)
    for k in range(2):
        sel = mat == k
        mu, lam = orc.lame(mats[k].E, mats[k].nu)
        tp = np.array([orc.hencky_tau(F[p].reshape(3, 3), mu, lam).ravel() for p in np.nonzero(sel)[0]])
        lhs = (un.V_ck[k][:, None] * un.tau_ck[k]).sum(0)
        rhs = (vol[sel][:, None] * tp).sum(0)
        assert np.allclose(lhs, rhs, rtol=1e-11, atol=1e-12 * np.abs(rhs).max())
        assert un.V_ck[k].sum() == pytest.approx(vol[sel].sum(), rel=1e-13)
    assert un.m_i.sum() == pytest.approx(mp.sum(), rel=1e-13)
    assert np.allclose((un.m_i[:, None] * un.v_i).sum(0), (mp[:, None] * v).sum(0), rtol=1e-11, atol=1e-13)


def test_unload_affine_reproduction(orc):
    """v_p = A x_p + b with G_p = A reproduces v_c = A x_c + b and G_c = A at every quadrature point,
    and v_i = A x_i + b at every node (APIC affine consistency of Eqs. p2c-mv-affine)."""
    n, x, _, F, _, vol, mat, mats = small_scene(seed=3)
    rng = np.random.default_rng(9)
    A, b = rng.normal(size=(3, 3)), rng.normal(size=3)
    v = x @ A.T + b
    G = np.tile(A.ravel(), (x.shape[0], 1))
    g = orc.Grid((n,) * 3, 1 / n)
    un = orc.unload(g, mats, x, v, F, G, vol, mat)
    act = un.m_c > 0
    xc = (g.cell_ijk() + 0.5) * g.dx
    assert np.allclose(un.v_c[act], xc[act] @ A.T + b, atol=1e-12)
    assert np.allclose(un.G_c[act], A.ravel()[None], atol=1e-12)
    an = un.m_i > 0
    xi = g.node_ijk() * g.dx
    assert np.allclose(un.v_i[an], xi[an] @ A.T + b, atol=1e-12)


def test_unload_single_particle_at_centre(orc):
    ex = GOLD["single_particle_at_centre"]
    g = orc.Grid((8, 8, 8), 1 / 8)
    x = np.array([[3.5, 4.5, 2.5]]) / 8
    v = np.array([ex["v_p"]])
    mats = [scenes.Material(1e4, 0.3, 1000.0)]
    un = orc.unload(g, mats, x, v, np.eye(3).reshape(1, 9), np.zeros((1, 9)), np.array([1e-3]),
                    np.zeros(1, np.int32))
    c = (3 * 8 + 4) * 8 + 2
    assert np.count_nonzero(un.m_c) == 1 and un.m_c[c] == pytest.approx(1.0)
    assert np.allclose(un.v_c[c], ex["v_p"])
    nz = np.nonzero(un.m_i)[0]
    assert len(nz) == 8
    assert np.allclose(un.m_i[nz], ex["node_mass_fraction"] * 1.0)
    assert np.allclose(un.v_i[nz], ex["v_p"])


def test_outside_domain_raises(orc):
    g = orc.Grid((8, 8, 8), 1 / 8)
    mats = [scenes.Material(1e4, 0.3, 1000.0)]
    with pytest.raises(ValueError):
        orc.unload(g, mats, np.array([[0.01, 0.5, 0.5]]), np.zeros((1, 3)), np.eye(3).reshape(1, 9),
                   np.zeros((1, 9)), np.array([1e-3]), np.zeros(1, np.int32))


# ------------------------------------------------------------------ C8 load
def _load_setup(orc, seed=11):
    n, x, v, F, G, vol, mat, mats = small_scene(seed=seed, prestrain=True)
    g = orc.Grid((n,) * 3, 1 / n)
    un = orc.unload(g, mats, x, v, F, G, vol, mat)
    return g, un, x, v, F, G


def test_load_uniform_and_affine(orc):
    """uniform nodal field -> v_p = c, G_p = 0, F unchanged; S:193 / P:1050 identity
    sum_i (x_i - x_c) (x) grad w_ic = I: affine nodal field v_i = A x_i + b -> G_p = A, v_p = A x_p + b."""
    g, un, x, v, F, G = _load_setup(orc)
    dt = 1e-3
    c = np.array([0.3, -0.2, 0.1])
    vi = np.tile(c, (g.nnodes, 1))
    x1, v1, F1, G1 = orc.g2p(g, dt, un.m_c, vi, x, v, F, G)
    assert np.allclose(v1, c, atol=1e-14) and np.allclose(G1, 0, atol=1e-12)
    assert np.allclose(F1, F, atol=1e-14) and np.allclose(x1, x + dt * c, atol=1e-15)
    rng = np.random.default_rng(1)
    A, b = rng.normal(size=(3, 3)), rng.normal(size=3)
    vi = (g.node_ijk() * g.dx) @ A.T + b
    x1, v1, F1, G1 = orc.g2p(g, dt, un.m_c, vi, x, v, F, G)
    assert np.allclose(G1, A.ravel()[None], atol=1e-11)
    assert np.allclose(v1, x @ A.T + b, atol=1e-12)
    Fn = np.einsum("ab,pbc->pac", np.eye(3) + dt * A, F.reshape(-1, 3, 3)).reshape(-1, 9)
    assert np.allclose(F1, Fn, atol=1e-13)


def test_load_hourglass_null_space(orc):
    """P:702 (Sec. 7): the trilinear hourglass modes lie in the null space of N2C — v_c = G_c = 0,
    so particles see nothing.  All 4 hourglass sign patterns x 3 components."""
    g, un, x, v, F, G = _load_setup(orc, seed=12)
    ijk = g.node_ijk()
    modes = [(ijk[:, 0] + ijk[:, 1]), (ijk[:, 1] + ijk[:, 2]), (ijk[:, 0] + ijk[:, 2]),
             (ijk[:, 0] + ijk[:, 1] + ijk[:, 2])]
    for m in modes:
        s = np.where(m % 2 == 0, 1.0, -1.0)
        for a in range(3):
            vi = np.zeros((g.nnodes, 3))
            vi[:, a] = s
            x1, v1, F1, G1 = orc.g2p(g, 1e-3, un.m_c, vi, x, v, F, G)
            assert np.allclose(v1, 0, atol=1e-14) and np.allclose(G1, 0, atol=1e-12)
    # a non-hourglass checkerboard along one axis is NOT filtered (sanity: the test can fail)
    vi = np.zeros((g.nnodes, 3))
    vi[:, 0] = np.where(ijk[:, 0] % 2 == 0, 1.0, -1.0)
    _, _, _, G1 = orc.g2p(g, 1e-3, un.m_c, vi, x, v, F, G)
    assert np.abs(G1).max() > 1.0


def test_grad_w_worked_example(orc):
    """dx=1, x_i - x_c = (1/2,1/2,1/2) -> grad w = (1/4,1/4,1/4).  Probed through G2P:
    a nodal field equal to e_a at ONE node of a single active cell gives G_c[a,:] = grad w_ic."""
    ex = GOLD["q1_grad_center_to_node"]
    g = orc.Grid((4, 4, 4), ex["dx"])
    m_c = np.zeros(g.ncells)
    c = (1 * 4 + 1) * 4 + 1
    m_c[c] = 1.0
    vi = np.zeros((g.nnodes, 3))
    node = (2 * 5 + 2) * 5 + 2  # the (+,+,+) corner of cell (1,1,1)
    vi[node, 0] = 1.0
    xp = np.array([[1.5, 1.5, 1.5]])  # particle at the centre: weight 1 on the cell
    _, v1, _, G1 = orc.g2p(g, 1e-3, m_c, vi, xp, np.zeros((1, 3)), np.eye(3).reshape(1, 9), np.zeros((1, 9)))
    assert np.allclose(G1[0, 0:3], ex["expected"], atol=1e-15)
    assert np.allclose(v1[0], [GOLD["center_to_node_weight_3d"]["expected"], 0, 0], atol=1e-15)
