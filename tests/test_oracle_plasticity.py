"""Oracle pins for fixed-point plasticity (PAPER §6.5).

The von Mises return map in Hencky space written as a right factor F^E = F P:
identity inside the yield surface and for volumetric trials, radial projection onto
||2 mu dev e|| = sqrt(2/3) sigma_y with the volume kept, objectivity and isotropy.  Inside Newton the
bases are re-projected at every iterate (S = S_base P, A(v) S = Z(A(v) S_base)) and held through the
iteration's PCG: the converged state is a fixed point (A(v*) S* = Z(A(v*) S_base), g(v*; S*) ~ 0),
every plastic slot ends inside the yield surface, an unreachable yield stress reproduces the elastic
solve bit for bit, and gradient / HVP with a (non-symmetric) plastic base match central differences.
Load return-maps the particles' trial F with the same map."""
import dataclasses

import numpy as np
import pytest

from paper_2602_07853_b200 import scenes

from .test_oracle_solver import elastic_part, make_scene

R23 = np.sqrt(2.0 / 3.0)


def hencky_dev_norm(F):
    C = F.T @ F
    e = 0.5 * np.log(np.linalg.eigvalsh(C))
    return np.linalg.norm(e - e.mean()), e.sum()


def rot(rng):
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return Q * np.sign(np.linalg.det(Q))


def test_inside_and_volumetric_are_identity(orc):
    mu, sy = 1.0, 0.1
    F = np.diag(np.exp([0.01, -0.005, 0.0]))  # 2 mu |e_dev| ~ 0.025 < sqrt(2/3) 0.1
    P, proj = orc.vm_plastic_P(F, mu, sy)
    assert not proj and np.array_equal(P, np.eye(3))
    rng = np.random.default_rng(1)
    R = rot(rng)
    Fv = 1.3 * R  # pure volumetric trial (all principal stretches equal)
    assert np.allclose(orc.vm_return(Fv, mu, 1e-6), Fv, atol=1e-12)


def test_spec_example_projects_onto_yield_surface(orc):
    """mu = 1, sigma_y = 0.1, trial deviatoric Hencky norm 0.5 -> post-projection deviatoric
    stress norm sigma_y sqrt(2/3) to 1e-10; the trace of e (the volume) is unchanged."""
    mu, sy = 1.0, 0.1
    d = np.array([1.0, -0.3, -0.7])
    d = 0.5 * d / np.linalg.norm(d - d.mean())
    e = d - d.mean() + 0.04  # |e_dev| = 0.5, tr e = 0.12
    rng = np.random.default_rng(2)
    R, Q = rot(rng), rot(rng)
    F = R @ np.diag(np.exp(e)) @ Q.T
    nrm, tr = hencky_dev_norm(F)
    assert nrm == pytest.approx(0.5, rel=1e-12)
    FE = orc.vm_return(F, mu, sy)
    nrmE, trE = hencky_dev_norm(FE)
    assert abs(2 * mu * nrmE - R23 * sy) <= 1e-10
    assert trE == pytest.approx(tr, abs=1e-12)
    assert np.linalg.det(FE) == pytest.approx(np.linalg.det(F), rel=1e-12)


def test_radial_direction_objectivity_isotropy(orc):
    rng = np.random.default_rng(3)
    mu, sy = 2.0, 0.05
    for _ in range(10):
        F = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
        if np.linalg.det(F) <= 0.1:
            continue
        FE = orc.vm_return(F, mu, sy)
        # radial: the projected deviatoric Hencky strain is parallel to the trial one (same eigenbasis)
        bt, be = F @ F.T, FE @ FE.T
        wt, Ut = np.linalg.eigh(bt)
        et = 0.5 * np.log(wt)
        ee = 0.5 * np.log(np.einsum("ia,ij,ja->a", Ut, be, Ut))  # be diagonal in the trial basis
        assert np.allclose(Ut.T @ be @ Ut, np.diag(np.exp(2 * ee)), atol=1e-10 * np.abs(be).max())
        dt_, de = et - et.mean(), ee - ee.mean()
        assert np.allclose(np.cross(dt_, de), 0.0, atol=1e-10)
        assert dt_ @ de > 0
        R, Q = rot(rng), rot(rng)
        assert np.allclose(orc.vm_return(R @ F, mu, sy), R @ FE, atol=1e-11)  # objectivity
        assert np.allclose(orc.vm_return(F @ Q, mu, sy), FE @ Q, atol=1e-11)  # isotropy


def plastic_scene(sy=150.0, seed=4, nmat=1, **kw):
    sc = make_scene(E=1e4, nu=0.3, vel=0.3, seed=seed, nmat=nmat, **kw)
    mats = [dataclasses.replace(m, yield_stress=sy if k == 0 else 0.0) for k, m in enumerate(sc.materials)]
    sc = dataclasses.replace(sc, materials=mats)
    return sc


def test_newton_fixed_point_and_yield_condition(orc):
    sc = plastic_scene()
    un, S, prob, v0 = orc.prepare(sc)
    _, nproj0 = prob.plastic_update(v0)
    assert nproj0 > 10  # the prestrain puts many slots outside the yield surface
    vN, st = prob.newton(v0, scenes.SolverCfg(eps_cg=1e-12, eps_newton=1e-10, newton_max=30))
    assert st["converged"] == 1
    Sst, _ = prob.plastic_update(vN)
    g = prob.with_bases(Sst).gradient(vN)
    g0 = prob.with_bases(prob.plastic_update(v0)[0]).gradient(v0)
    fr = prob.freed != 0
    assert np.linalg.norm(g[fr]) <= 1e-9 * np.linalg.norm(g0[fr])
    # every slot's elastic state A(v*) S* = Z(A(v*) S_base) is inside (or on) the yield surface
    mu = sc.materials[0].E / (2 * (1 + sc.materials[0].nu))
    grid = prob.grid
    ijk = grid.cell_ijk()
    n1 = grid.n[1] + 1
    for c in np.nonzero(un.V_ck[0] > 0)[0][:200]:
        ci = ijk[c]
        corners = [((ci[0] + ((o >> 2) & 1)) * n1 + ci[1] + ((o >> 1) & 1)) * n1 + ci[2] + (o & 1) for o in range(8)]
        gw = np.array([[((o >> 2) & 1) - 0.5, ((o >> 1) & 1) - 0.5, (o & 1) - 0.5] for o in range(8)]) / (2 * grid.dx)
        G = sum(np.outer(vN[corners[o]], gw[o]) for o in range(8))
        A = np.eye(3) + sc.dt * G
        FE = A @ Sst[0, c].reshape(3, 3)
        assert np.allclose(FE, orc.vm_return(A @ S[0, c].reshape(3, 3), mu, 150.0), atol=1e-12)
        nrm, _ = hencky_dev_norm(FE)
        assert 2 * mu * nrm <= R23 * 150.0 * (1 + 1e-9)


def test_unreachable_yield_is_the_elastic_solve(orc):
    sc_el = make_scene(E=1e4, nu=0.3, vel=0.3, seed=4)
    sc_pl = plastic_scene(sy=1e30)
    _, _, p_el, v0 = orc.prepare(sc_el)
    _, _, p_pl, v0p = orc.prepare(sc_pl)
    cfg = scenes.SolverCfg(eps_cg=1e-12, eps_newton=1e-10)
    va, sa = p_el.newton(v0, cfg)
    vb, sb = p_pl.newton(v0p, cfg)
    assert np.array_equal(va, vb) and sa["cg_iters"] == sb["cg_iters"]


def test_gradient_hvp_fd_with_plastic_base(orc):
    """With the iterate's (non-symmetric) base S = S_base P held fixed: g = dPhi/dv and H u = dg/dv u by
    central differences; H symmetric."""
    sc = plastic_scene(seed=6)
    un, S, prob, v0 = orc.prepare(sc)
    Sk, n = prob.plastic_update(v0)
    assert n > 0
    Sm = Sk[0][un.V_ck[0] > 0].reshape(-1, 3, 3)
    assert np.abs(Sm - Sm.transpose(0, 2, 1)).max() > 1e-6  # really non-symmetric
    pk = prob.with_bases(Sk)
    rng = np.random.default_rng(7)
    act = (prob.m_i > 0)[:, None]
    v = v0 + 0.01 * rng.normal(size=v0.shape) * act
    g = pk.gradient(v)
    h = 1e-6
    nodes = np.nonzero(act[:, 0])[0]
    for i in rng.choice(nodes, 15, replace=False):
        for a in range(3):
            vp, vm = v.copy(), v.copy()
            vp[i, a] += h
            vm[i, a] -= h
            fd = (pk.energy(vp) - pk.energy(vm)) / (2 * h)
            assert fd == pytest.approx(g[i, a], rel=1e-5, abs=1e-7 * np.abs(g).max())
    u = rng.normal(size=v.shape) * act
    w = rng.normal(size=v.shape) * act
    Hu = pk.hvp(v, u)
    fdH = (pk.gradient(v + h * u) - pk.gradient(v - h * u)) / (2 * h)
    assert np.linalg.norm(fdH - Hu) <= 1e-6 * np.linalg.norm(Hu)
    assert abs((w * Hu).sum() - (u * pk.hvp(v, w)).sum()) <= 1e-11 * abs((w * Hu).sum())


def test_load_return_maps_plastic_particles(orc):
    sc = plastic_scene(sy=100.0, nmat=2)
    r = orc.step(sc)
    mu = sc.materials[0].E / (2 * (1 + sc.materials[0].nu))
    F = r.particles[2].reshape(-1, 3, 3)
    pl = sc.mat == 0
    norms = np.array([hencky_dev_norm(f)[0] for f in F[pl]])
    assert np.all(2 * mu * norms <= R23 * 100.0 * (1 + 1e-9))
    # the elastic material's particles are not projected: some exceed that yield stress
    normsE = np.array([hencky_dev_norm(f)[0] for f in F[~pl]])
    mu1 = sc.materials[1].E / (2 * (1 + sc.materials[1].nu))
    assert np.any(2 * mu1 * normsE > R23 * 100.0)
