"""Oracle pins, part 3: incremental potential, gradient, HVP, Jacobi diagonal (C6) and the
Newton-PCG step (C7).

Pins: central finite differences, Hessian symmetry, e.H.e diagonal, the
constant-strain patch test, rigid rotation, the textbook one-point linear hex
stiffness at S=I, G=0, the explicit-force special case, brute-force dense solves,
mass-only and zero-stress limits, the O(dt^2) stiff limit.
"""
import dataclasses

import numpy as np
import pytest

from paper_2602_07853_b200 import scenes


def make_scene(n=8, lo=2, hi=6, E=1e8, nu=0.3, rho=1000.0, dt=1e-3, prestrain=True, vel=0.3, seed=0,
               lattice=False, nmat=1, gravity=scenes.GRAVITY, boxes=(), kind=0):
    cells = scenes.cells_box([lo] * 3, [hi] * 3)
    if lattice:  # unjittered: sub-cell centres
        k = 2
        s = scenes.cells_box([0, 0, 0], [k, k, k]).astype(float)
        x = ((cells[:, None, :] + (s[None] + 0.5) / k) / n).reshape(-1, 3)
    else:
        x = scenes.stratified(cells, n, 2, seed=seed)
    rng = np.random.default_rng(seed + 1)
    v = vel * rng.normal(size=x.shape)
    F = scenes._prestrain(x.shape[0], seed + 3) if prestrain else np.tile(np.eye(3).ravel(), (x.shape[0], 1))
    mat = rng.integers(0, nmat, size=x.shape[0]).astype(np.int32)
    # kind: 0 StVK-Hencky, 1 split Neo-Hookean, 2 water; "mix": Hencky + Neo-Hookean slots,
    # "wmix": Hencky + water slots (material slots k = 0, 1)
    if kind == "mix":
        kinds = [k % 2 for k in range(nmat)]
    elif kind == "wmix":
        kinds = [2 * (k % 2) for k in range(nmat)]
    else:
        kinds = [kind] * nmat
    mats = [scenes.Material(E * (1 + 0.7 * k), nu, rho, kinds[k]) for k in range(nmat)]
    return scenes.Scene(name="t", precision=64, n=(n, n, n), dx=1 / n, dt=dt, materials=mats, x=x, v=v, F=F,
                        G=np.zeros((x.shape[0], 9)), vol=np.full(x.shape[0], (1 / n) ** 3 / 8), mat=mat,
                        dirichlet=list(boxes), solver=scenes.SolverCfg(eps_cg=1e-12, eps_newton=1e-10),
                        gravity=gravity)


def elastic_part(prob, g_or_hu, v_or_u, vhat=None):
    m = prob.m_i[:, None]
    if vhat is None:
        return g_or_hu - m * v_or_u
    return g_or_hu - m * (v_or_u - vhat)


# ------------------------------------------------------------------ C6 derivatives
@pytest.mark.parametrize("nmat,kind", [(1, 0), (2, 0), (1, 1), (2, "mix"), (1, 2), (2, "wmix")])
def test_gradient_matches_fd(orc, nmat, kind):
    sc = make_scene(nmat=nmat, kind=kind)
    un, S, prob, v0 = orc.prepare(sc)
    rng = np.random.default_rng(5)
    act = prob.m_i > 0
    v = v0 + 0.01 * rng.normal(size=v0.shape) * act[:, None]  # seed-5 style probe
    g = prob.gradient(v)
    gel = elastic_part(prob, g, v, prob.vhat)
    h = 1e-6
    fd = np.zeros_like(v)
    for i in np.nonzero(act)[0]:
        for a in range(3):
            vp, vm = v.copy(), v.copy()
            vp[i, a] += h
            vm[i, a] -= h
            fd[i, a] = (prob.energy(vp) - prob.energy(vm)) / (2 * h)
    fdel = elastic_part(prob, fd, v, prob.vhat)
    assert np.linalg.norm(gel) > 0.1 * np.linalg.norm(g)  # elastic part is not negligible
    assert np.linalg.norm(fd - g) <= 1e-6 * np.linalg.norm(g)
    assert np.linalg.norm(fdel - gel) <= 1e-5 * np.linalg.norm(gel)


@pytest.mark.parametrize("nmat,kind", [(1, 0), (2, 0), (1, 1), (2, "mix"), (1, 2), (2, "wmix")])
def test_hvp_matches_fd_and_is_symmetric(orc, nmat, kind):
    sc = make_scene(nmat=nmat, seed=2, kind=kind)
    un, S, prob, v0 = orc.prepare(sc)
    rng = np.random.default_rng(4)
    act = (prob.m_i > 0)[:, None]
    v = v0 + 0.01 * rng.normal(size=v0.shape) * act
    u = rng.normal(size=v0.shape) * act
    w = rng.normal(size=v0.shape) * act
    Hu = prob.hvp(v, u)
    h = 1e-6
    fd = (prob.gradient(v + h * u) - prob.gradient(v - h * u)) / (2 * h)
    el, fdel = elastic_part(prob, Hu, u), elastic_part(prob, fd, u)
    assert np.linalg.norm(el) > 0.5 * np.linalg.norm(prob.m_i[:, None] * u)
    assert np.linalg.norm(fdel - el) <= 1e-6 * np.linalg.norm(el)
    Hw = prob.hvp(v, w)
    assert abs((u * Hw).sum() - (w * Hu).sum()) <= 1e-12 * abs((u * Hw).sum())


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_diag_is_eHe(orc, kind):
    sc = make_scene(seed=3, kind=kind)
    un, S, prob, v0 = orc.prepare(sc)
    rng = np.random.default_rng(6)
    v = v0 + 0.01 * rng.normal(size=v0.shape) * (prob.m_i > 0)[:, None]
    D = prob.diag(v)
    nodes = np.nonzero(prob.m_i > 0)[0]
    for i in rng.choice(nodes, 12, replace=False):
        for a in range(3):
            e = np.zeros_like(v)
            e[i, a] = 1.0
            assert D[i, a] == pytest.approx(prob.hvp(v, e)[i, a], rel=1e-12)


# both solid laws linearise to 2 mu eps + lam tr(eps) I at rest; water to kappa tr(eps) I
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_textbook_linear_hex_stiffness(orc, kind):
    """At S = I and v = 0 (G = 0, A = I): K_c = dt^2 V C with C:e = 2 mu sym(e) + lam tr(e) I, the
    one-point trilinear-hex linear-elastic stiffness."""
    sc = make_scene(prestrain=False, vel=0.0, seed=7, kind=kind)
    un, S, prob, v0 = orc.prepare(sc)
    g = prob.grid
    rng = np.random.default_rng(8)
    u = rng.normal(size=(g.nnodes, 3)) * (prob.m_i > 0)[:, None]
    v = np.zeros_like(u)
    Hu = prob.hvp(v, u)
    mu, lam = orc.lame(sc.materials[0].E, sc.materials[0].nu)
    if kind == 2:
        mu, lam = 0.0, sc.materials[0].E  # psi = kappa/2 (J-1)^2, kappa = E
    ref = prob.m_i[:, None] * u
    ijk = g.cell_ijk()
    n1 = g.n[1] + 1
    for c in np.nonzero(un.m_c > 0)[0]:
        ci = ijk[c]
        corners = [((ci[0] + ((o >> 2) & 1)) * n1 + ci[1] + ((o >> 1) & 1)) * n1 + ci[2] + (o & 1) for o in range(8)]
        gw = np.array([[((o >> 2) & 1) - 0.5, ((o >> 1) & 1) - 0.5, (o & 1) - 0.5] for o in range(8)]) / (2 * g.dx)
        dG = sum(np.outer(u[corners[o]], gw[o]) for o in range(8))
        sig = 2 * mu * 0.5 * (dG + dG.T) + lam * np.trace(dG) * np.eye(3)
        P = sc.dt ** 2 * un.V_ck[0, c] * sig
        for o in range(8):
            ref[corners[o]] += P @ gw[o]
    assert np.allclose(Hu, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_explicit_force_special_case(orc):
    """At G_c(v) = 0 (v = 0): g = m (0 - vhat) + dt sum V tau(S) grad w = -m vhat - dt f^n, with f^n the
    explicit force of Eq. explicitforce, because tau(S_c) = tau_c (Eq. rotfree-def)."""
    sc = make_scene(seed=9, nmat=2)
    un, S, prob, v0 = orc.prepare(sc)
    v = np.zeros_like(v0)
    g = prob.gradient(v)
    f = orc.explicit_force(prob.grid, 2, un.m_c, un.V_ck, un.tau_ck)
    ref = -prob.m_i[:, None] * prob.vhat - sc.dt * f
    assert np.allclose(g, ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
    assert np.abs(f).max() > 0


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_patch_test_affine_zero_interior_force(orc, kind):
    """Constant-strain patch test (north_star): unjittered lattice -> interior V_c = dx^3 exactly;
    uniform F_p -> uniform S; affine v -> zero net elastic force on interior nodes (sum_c grad w_ic = 0)."""
    n = 12
    sc = make_scene(n=n, lo=2, hi=10, lattice=True, prestrain=False, seed=1, kind=kind)
    F0 = np.array([[1.05, 0.02, 0.0], [0.01, 0.97, 0.03], [0.0, -0.02, 1.01]])
    sc = dataclasses.replace(sc, F=np.tile(F0.ravel(), (sc.x.shape[0], 1)))
    un, S, prob, v0 = orc.prepare(sc)
    g = prob.grid
    ijk_c = g.cell_ijk()
    interior_c = np.all((ijk_c >= 3) & (ijk_c <= 8), axis=1)
    assert np.allclose(un.V_ck[0][interior_c], g.dx ** 3, rtol=1e-14)
    Sact = S[0][un.m_c > 0]
    assert np.allclose(Sact, Sact[0][None], atol=1e-13)
    A = np.array([[0.3, -0.2, 0.1], [0.05, 0.1, 0.4], [-0.3, 0.2, -0.1]])
    v = (g.node_ijk() * g.dx) @ A.T * (prob.m_i > 0)[:, None]
    gel = elastic_part(prob, prob.gradient(v), v, prob.vhat)
    ijk_n = g.node_ijk()
    interior_n = np.all((ijk_n >= 4) & (ijk_n <= 8), axis=1)  # all 8 adjacent cells in 3..8
    boundary = (prob.m_i > 0) & ~interior_n
    assert np.abs(gel[interior_n]).max() <= 1e-12 * np.abs(gel[boundary]).max()
    assert np.abs(gel[boundary]).max() > 0


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_rigid_rotation(orc, kind):
    """v_i = ((R - I)/dt)(x_i - x0) gives G_c = (R - I)/dt exactly, F = R S: with S = I the elastic
    energy and force vanish; with S != I the elastic energy equals that at v = 0 (isotropy)."""
    ang = 0.3
    R = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1.0]])
    for prestrain in (False, True):
        sc = make_scene(prestrain=prestrain, seed=4, kind=kind)
        un, S, prob, v0 = orc.prepare(sc)
        g = prob.grid
        x0 = np.array([0.5, 0.5, 0.5])
        v = ((g.node_ijk() * g.dx - x0) @ (R - np.eye(3)).T / sc.dt) * (prob.m_i > 0)[:, None]
        inertia = lambda vv: 0.5 * (prob.m_i[:, None] * (vv - prob.vhat) ** 2).sum()
        Eel_rot = prob.energy(v) - inertia(v)
        Eel_0 = prob.energy(np.zeros_like(v)) - inertia(np.zeros_like(v))
        if not prestrain:
            assert abs(Eel_rot) <= 1e-12 * inertia(v)
            gel = elastic_part(prob, prob.gradient(v), v, prob.vhat)
            assert np.abs(gel).max() <= 1e-9 * np.abs(prob.m_i[:, None] * v).max()
        else:
            assert Eel_rot == pytest.approx(Eel_0, rel=1e-10)
            assert Eel_0 > 0


# ------------------------------------------------------------------ C7 Newton-PCG
def test_zero_stress_uniform_velocity(orc):
    """zero stress, no gravity, uniform velocity -> v^{n+1} = v^n with no Newton work."""
    sc = make_scene(prestrain=False, vel=0.0, gravity=(0.0, 0.0, 0.0))
    sc = dataclasses.replace(sc, v=np.tile([0.2, -0.1, 0.05], (sc.x.shape[0], 1)))
    r = orc.step(sc)
    act = r.problem.m_i > 0
    # the gradient at v^n is rounding noise only (~1e-16 relative), so Newton has nothing to do
    assert r.stats["grad_norm0"] <= 1e-12 * np.linalg.norm(r.problem.m_i[:, None] * r.v_new)
    assert np.allclose(r.v_new[act], [0.2, -0.1, 0.05], atol=1e-13)


def test_mass_only_limit(orc):
    """E -> 0: H = M = Jacobi diagonal, so one PCG iteration gives v = vhat = v^n + dt g."""
    sc = make_scene(E=1e-9, prestrain=False, vel=0.3)
    r = orc.step(sc)
    act = r.problem.m_i > 0
    assert r.stats["cg_iters"][0] == 1
    assert np.allclose(r.v_new[act], r.problem.vhat[act], atol=1e-12)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_newton_bruteforce_dense(orc, kind):
    """Brute force on a tiny grid: dense H from n HVPs is symmetric positive definite; one Newton
    iteration with exact PCG equals v + H^{-1}(-g) (dense Cholesky); the converged step has ||g|| ~ 0
    and the energy decreases at every accepted iterate."""
    sc = make_scene(n=6, lo=2, hi=4, E=1e7, seed=5, boxes=[scenes.DirichletBox((-1, -1, -1), (2, 2 / 6, 2), (0, 0, 0))],
                    kind=kind)
    un, S, prob, v0 = orc.prepare(sc)
    fr = np.nonzero(prob.freed)[0]
    assert 0 < len(fr) < np.count_nonzero(prob.m_i)
    dofs = [(i, a) for i in fr for a in range(3)]
    H = np.zeros((len(dofs), len(dofs)))
    for j, (i, a) in enumerate(dofs):
        e = np.zeros_like(v0)
        e[i, a] = 1.0
        Hu = prob.hvp(v0, e)
        H[:, j] = [Hu[ii, aa] for ii, aa in dofs]
    assert np.allclose(H, H.T, rtol=0, atol=1e-12 * np.abs(H).max())
    L = np.linalg.cholesky(0.5 * (H + H.T))
    g = prob.gradient(v0)
    gf = np.array([g[i, a] for i, a in dofs])
    p = np.linalg.solve(H, -gf)
    solver = scenes.SolverCfg(eps_cg=1e-14, eps_newton=1e-30, newton_max=1, cg_max=10 * len(dofs))
    v1, st = prob.newton(v0, solver)
    assert st["ls_iters"][0] == 0
    got = np.array([v1[i, a] - v0[i, a] for i, a in dofs])
    assert np.allclose(got, p, rtol=1e-9, atol=1e-11 * np.abs(p).max())
    fixed = (prob.m_i > 0) & (prob.freed == 0)
    assert np.array_equal(v1[fixed], v0[fixed])
    # full solve
    solver = scenes.SolverCfg(eps_cg=1e-10, eps_newton=1e-10, newton_max=20)
    vN, st = prob.newton(v0, solver)
    assert st["converged"] == 1
    gN = prob.gradient(vN)
    assert np.linalg.norm(gN[fr]) <= 1e-10 * np.linalg.norm(g[fr])
    assert prob.energy(vN) < prob.energy(v0)
    # energies along iterates are monotone
    e_prev, v = prob.energy(v0), v0
    for k in range(st["newton_iters"]):
        v, _ = prob.newton(v, dataclasses.replace(solver, newton_max=1))
        e = prob.energy(v)
        assert e <= e_prev + 1e-12 * abs(e_prev)
        e_prev = e


def test_stiff_limit_dt2(orc):
    """implicit and explicit updates agree to O(dt^2) as dt -> 0 (error ratio ~4 per halving)."""
    errs = []
    for dt in (1e-3, 5e-4, 2.5e-4, 1.25e-4):
        sc = make_scene(E=1e5, seed=6, dt=dt)
        un, S, prob, v0 = orc.prepare(sc)
        vN, st = prob.newton(v0, scenes.SolverCfg(eps_cg=1e-13, eps_newton=1e-12, newton_max=20))
        act = prob.m_i > 0
        f = orc.explicit_force(prob.grid, 1, un.m_c, un.V_ck, un.tau_ck)
        vex = np.where(act[:, None], prob.vhat + dt * f / np.where(act, prob.m_i, 1.0)[:, None], 0.0)
        errs.append(np.linalg.norm((vN - vex)[act]))
    ratios = [errs[i] / errs[i + 1] for i in range(3)]
    assert all(r > 3.0 for r in ratios) and 3.6 < ratios[-1] < 4.4, ratios  # log2 slope -> 2


# ---- orc_dirichlet (amb-9: node i is prescribed when lo <= x_i <= hi on every axis) -------------------
def test_dirichlet_floor_worked_example():
    """Hand count on an 8^3 grid (dx = 1/8, exact in binary): the cfg4 / cfg5 floor "nodes with y <= 3 dx"
    prescribes exactly the node planes j = 0, 1, 2, 3 (9 x 4 x 9 = 324 nodes; the plane at y = 3 dx is
    included, y = 4 dx is not); nodes there with m_i = 0 are no DOF either; the box velocity is returned
    for every prescribed node, 0 elsewhere."""
    import oracle
    grid = oracle.Grid((8, 8, 8), 1 / 8)
    inf = float("inf")
    boxes = [scenes.DirichletBox((-inf, -inf, -inf), (inf, 3 / 8, inf), (0.5, -1.0, 2.0))]
    m_i = np.ones(grid.nnodes)
    m_i[oracle.Grid((8, 8, 8), 1 / 8).node_ijk()[:, 0] == 8] = 0.0  # the x = 1 plane carries no mass
    freed, vfix = oracle.dirichlet(grid, boxes, m_i)
    ijk = grid.node_ijk()
    fixed = np.all(vfix == [0.5, -1.0, 2.0], axis=1)
    assert fixed.sum() == 9 * 4 * 9
    assert set(np.unique(ijk[fixed, 1]).tolist()) == {0, 1, 2, 3}
    assert np.all(vfix[~fixed] == 0.0)
    # free DOFs: m_i > 0 and j >= 4 -> x-planes 0..7 (8) x y-planes 4..8 (5) x 9
    assert freed.sum() == 8 * 5 * 9
    assert np.all(freed[ijk[:, 1] <= 3] == 0) and np.all(freed[ijk[:, 0] == 8] == 0)


def test_dirichlet_first_box_wins_and_plate():
    """Two overlapping boxes: a node inside both takes the FIRST box's velocity (the header's rule);
    the cfg5 plate "y >= top" with top on a node plane includes that plane.  Checked against a
    brute-force membership count over explicit integer node indices (no coordinates): on a 16^3 grid,
    floor = planes j <= 3, plate = planes j >= 12, a side box i <= 1 overlapping both."""
    import oracle
    n = 16
    grid = oracle.Grid((n, n, n), 1 / n)
    inf = float("inf")
    boxes = [scenes.DirichletBox((-inf, -inf, -inf), (inf, 3 / n, inf), (0.0, 0.0, 0.0)),
             scenes.DirichletBox((-inf, 12 / n, -inf), (inf, inf, inf), (0.0, -0.5, 0.0)),
             scenes.DirichletBox((-inf, -inf, -inf), (1 / n, inf, inf), (7.0, 7.0, 7.0))]
    freed, vfix = oracle.dirichlet(grid, boxes, np.ones(grid.nnodes))
    for idx, (i, j, k) in enumerate(grid.node_ijk()):
        want = (0.0, 0.0, 0.0) if j <= 3 else (0.0, -0.5, 0.0) if j >= 12 else (7.0, 7.0, 7.0) if i <= 1 else None
        assert freed[idx] == (want is None)
        assert tuple(vfix[idx]) == (want if want is not None else (0.0, 0.0, 0.0))


# ---- per-cell PSD projection of the Hessian (solver option psd, DESIGN.md §2 amb-6b) -----
def test_psd_project9_matches_eigh_clamp(orc):
    """The oracle's cyclic-Jacobi projection equals LAPACK's eigh with the negative eigenvalues clamped
    (an independent eigensolver), including repeated and zero eigenvalues."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        Q, _ = np.linalg.qr(rng.normal(size=(9, 9)))
        lam = rng.normal(size=9) * 10.0 ** rng.uniform(-3, 3)
        if trial % 4 == 1:
            lam[:3] = lam[0]  # repeated
        if trial % 4 == 2:
            lam[5] = 0.0
        M = (Q * lam) @ Q.T
        w, U = np.linalg.eigh(M)
        want = (U * np.maximum(w, 0.0)) @ U.T
        got = orc.psd_project9(M)
        assert np.allclose(got, got.T, rtol=0, atol=1e-13 * np.abs(M).max())
        assert np.abs(got - want).max() <= 1e-11 * np.abs(M).max()


def _compressed_scene(J=0.93, n=6):
    """A uniformly compressed block (F_p = J^{1/3} I): a hydrostatic Kirchhoff stress tau < 0 makes the
    rotation modes of K_c negative (geometric stiffness), so the exact Hessian is indefinite."""
    sc = make_scene(n=n, lo=2, hi=4, E=1e6, prestrain=False, vel=0.05, seed=3)
    F = np.tile((J ** (1 / 3) * np.eye(3)).ravel(), (sc.x.shape[0], 1))
    return dataclasses.replace(sc, F=F)


def _dense_elastic(prob, v0):
    fr = np.nonzero(prob.m_i > 0)[0]
    dofs = [(i, a) for i in fr for a in range(3)]
    H = np.zeros((len(dofs), len(dofs)))
    for j, (i, a) in enumerate(dofs):
        e = np.zeros_like(v0)
        e[i, a] = 1.0
        Hu = prob.hvp(v0, e) - prob.m_i[:, None] * e
        H[:, j] = [Hu[ii, aa] for ii, aa in dofs]
    return H, dofs


def test_psd_hessian_is_psd_and_dominates_exact(orc):
    """Compressed block: the exact elastic Hessian has negative eigenvalues; the projected one is
    symmetric PSD, H+ - H is PSD (clamping only adds sum |lambda_-| q q^T per cell), and the projected
    Jacobi diagonal is the diagonal of the dense projected Hessian."""
    sc = _compressed_scene()
    un, S, prob, v0 = orc.prepare(sc)
    H, dofs = _dense_elastic(prob, v0)
    Hp, _ = _dense_elastic(prob.with_psd(True), v0)
    scale = np.abs(H).max()
    assert np.linalg.eigvalsh(0.5 * (H + H.T)).min() < -1e-6 * scale
    assert np.allclose(Hp, Hp.T, rtol=0, atol=1e-11 * scale)
    assert np.linalg.eigvalsh(0.5 * (Hp + Hp.T)).min() >= -1e-10 * scale
    assert np.linalg.eigvalsh(0.5 * ((Hp - H) + (Hp - H).T)).min() >= -1e-10 * scale
    D = prob.with_psd(True).diag(v0)
    want = np.array([Hp[j, j] for j in range(len(dofs))]) + np.array([prob.m_i[i] for i, _ in dofs])
    got = np.array([D[i, a] for i, a in dofs])
    assert np.allclose(got, want, rtol=1e-12, atol=0)


def test_psd_is_identity_on_convex_cells(orc):
    """Stretched block (F_p = 1.05^{1/3} I, tension): every K_c is PSD already, so the projected HVP equals
    the exact one to rounding."""
    sc = _compressed_scene(J=1.05)
    un, S, prob, v0 = orc.prepare(sc)
    u = np.random.default_rng(4).normal(size=v0.shape) * (prob.m_i > 0)[:, None]
    h = prob.hvp(v0, u) - prob.m_i[:, None] * u
    hp = prob.with_psd(True).hvp(v0, u) - prob.m_i[:, None] * u
    assert np.linalg.norm(hp - h) <= 1e-10 * np.linalg.norm(h)


def test_psd_newton_converges_without_negative_curvature(orc):
    """Projected Newton on the compressed block: PCG never meets negative curvature and the step
    converges to the Newton tolerance on the true gradient."""
    sc = _compressed_scene()
    un, S, prob, v0 = orc.prepare(sc)
    solver = dataclasses.replace(sc.solver, psd=True, eps_newton=1e-9, eps_cg=1e-10)
    v, st = prob.newton(v0, solver)
    assert st["neg_curv"] == 0 and st["converged"] == 1
    assert np.linalg.norm(prob.gradient(v)[prob.freed == 1]) <= 1e-9 * st["grad_norm0"] * 1.0001
