"""GPU parity: the CUDA path (called through the C ABI) against the fp64 oracle on the same seeded
inputs.  Bars (BASELINE.json north_star): bit-exact indices / active-block lists; relative L2
<= 1e-10 (fp64) / 1e-5 (fp32) on unload, gradient, HVP; <= 1e-8 / 1e-4 after a full step."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2602_07853_b200 import scenes

from ._parity import TOL, Pair, cell_ids, node_ids, rel_l2

pytestmark = pytest.mark.gpu


def small_cfg2(precision=32, k=16):
    """cfg2's material / field / dt on a 32^3 grid with a k^3 block (oracle-sized)."""
    n = 32
    cells = scenes.cells_box([8] * 3, [8 + k] * 3)
    dt_ = np.float32 if precision == 32 else np.float64
    x = scenes.stratified(cells, n, 2, seed=0, dtype=dt_)
    v, G = scenes.eval_smooth_field(x, scenes.smooth_field(2))
    tol = (1e-8, 1e-9) if precision == 64 else (1e-5, 1e-5)
    return scenes._assemble("cfg2s", precision, n, 2e-3, [scenes.Material(1e5, 0.4, 1000.0)], x, v,
                            scenes._identity(x.shape[0], np.float64), G, np.zeros(x.shape[0], np.int32), 8, [],
                            scenes.SolverCfg(eps_cg=tol[0], eps_newton=tol[1], ls_slack=1e-13 if precision == 64 else 1e-6), 1)


def two_material(precision=64, kinds=(0, 0), yields=(0.0, 0.0)):
    """Two materials mixed in the same cells + a sticky floor (exercises slots and Dirichlet); kinds
    selects each material's law (0 StVK-Hencky, 1 split Neo-Hookean, 2 J-based water)."""
    n = 16
    cells = scenes.cells_box([4, 2, 4], [12, 10, 12])
    dt_ = np.float32 if precision == 32 else np.float64
    x = scenes.stratified(cells, n, 2, seed=0, dtype=dt_)
    rng = np.random.default_rng(1)
    v = rng.normal(0, 0.3, size=x.shape)
    F = scenes._prestrain(x.shape[0], 3)
    mat = rng.integers(0, 2, size=x.shape[0]).astype(np.int32)
    floor = scenes.DirichletBox((-1e9, -1e9, -1e9), (1e9, 3 / n, 1e9), (0.0, 0.0, 0.0))
    tol = (1e-8, 1e-9) if precision == 64 else (1e-5, 1e-5)
    return scenes._assemble("mix", precision, n, 1e-3,
                            [scenes.Material(1e5, 0.3, 1000.0, kinds[0], yields[0]),
                             scenes.Material(3e6, 0.45, 2500.0, kinds[1], yields[1])],
                            x, v, F,
                            np.zeros((x.shape[0], 9)), mat, 8, [floor],
                            scenes.SolverCfg(eps_cg=tol[0], eps_newton=tol[1]), 1)


def water_block(precision=64):
    """A water block (kind 2, kappa = E = 2e5) with J_p ~ U(0.97, 1.03) (F_p = J_p^{1/3} I),
    random velocities, over a sticky floor."""
    n = 16
    cells = scenes.cells_box([4, 2, 4], [12, 9, 11])
    dt_ = np.float32 if precision == 32 else np.float64
    x = scenes.stratified(cells, n, 2, seed=2, dtype=dt_)
    rng = np.random.default_rng(7)
    v = rng.normal(0, 0.3, size=x.shape)
    J = rng.uniform(0.97, 1.03, size=x.shape[0])
    F = (J[:, None] ** (1 / 3)) * np.eye(3).ravel()[None, :]
    floor = scenes.DirichletBox((-1e9, -1e9, -1e9), (1e9, 3 / n, 1e9), (0.0, 0.0, 0.0))
    tol = (1e-8, 1e-9) if precision == 64 else (1e-5, 1e-5)
    return scenes._assemble("water", precision, n, 1e-3, [scenes.Material(2e5, 0.0, 1000.0, 2)], x, v, F,
                            np.zeros((x.shape[0], 9)), np.zeros(x.shape[0], np.int32), 8, [floor],
                            scenes.SolverCfg(eps_cg=tol[0], eps_newton=tol[1]), 1)


def plastic_cube(precision=64):
    """cfg1b (pre-strained cube, E = 1e4) with von Mises sigma_y = 150 Pa: 2 mu |e_dev| of the prestrain
    (~400 Pa) puts most slots outside the yield surface."""
    sc = scenes.cfg1(prestrain=True, precision=precision)
    return dataclasses.replace(sc, materials=[dataclasses.replace(sc.materials[0], yield_stress=150.0)])


def compressed_cube(precision=64):
    """cfg1's cube uniformly compressed (F_p = 0.93^{1/3} R_p-free, tau < 0: the exact Hessian is indefinite)
    on a sticky floor, solved with the per-cell PSD-projected Hessian (solver psd)."""
    sc = scenes.cfg1(prestrain=False, precision=precision)
    F = np.tile((0.93 ** (1 / 3) * np.eye(3)).ravel(), (sc.x.shape[0], 1))
    floor = scenes.DirichletBox((-1e9, -1e9, -1e9), (1e9, 4.5 / 16, 1e9), (0.0, 0.0, 0.0))
    return dataclasses.replace(sc, name="psd", F=F, materials=[scenes.Material(1e6, 0.3, 1000.0)], dirichlet=[floor],
                               solver=dataclasses.replace(sc.solver, psd=True))


def compressing_cube(precision=32):
    """cfg1's cube at rest (F_p = I, so every stretch base S = I) with a converging velocity field v = -5 (x - c):
    the trial deformation compresses the cells and the exact Hessian turns indefinite; with the PSD-projected
    Hessian and S = I the fp32 path projects the compressed tangent blockwise (amb-6b)."""
    sc = scenes.cfg1(prestrain=False, precision=precision)
    v = -5.0 * (sc.x - 0.5)
    floor = scenes.DirichletBox((-1e9, -1e9, -1e9), (1e9, 4.5 / 16, 1e9), (0.0, 0.0, 0.0))
    return dataclasses.replace(sc, name="psdI", v=v, materials=[scenes.Material(1e6, 0.3, 1000.0)], dirichlet=[floor],
                               solver=dataclasses.replace(sc.solver, psd=True))


SCENES = {
    "cfg1": lambda: scenes.cfg1(),
    "cfg1b": lambda: scenes.cfg1(prestrain=True),
    "cfg1_fp32": lambda: dataclasses.replace(scenes.cfg1(prestrain=True, precision=32)),
    "cfg2s_fp32": lambda: small_cfg2(32),
    "cfg2s_fp64": lambda: small_cfg2(64),
    "mix_fp64": lambda: two_material(64),
    "mix_fp32": lambda: two_material(32),
    # split Neo-Hookean: alone (pre-strained cube) and mixed with StVK-Hencky in the same cells
    "nh_fp64": lambda: dataclasses.replace(scenes.cfg1(prestrain=True),
                                           materials=[scenes.Material(1e4, 0.3, 1000.0, 1)]),
    "lawmix_fp64": lambda: two_material(64, (0, 1)),
    "lawmix_fp32": lambda: two_material(32, (1, 0)),
    # J-based water: alone, and water + StVK-Hencky in the same cells (sand-and-water shape)
    "water_fp64": lambda: water_block(64),
    "watermix_fp64": lambda: two_material(64, (0, 2)),
    "watermix_fp32": lambda: two_material(32, (2, 0)),
    # fixed-point von Mises plasticity: pre-strained cube past the yield surface, and a
    # plastic + elastic mixture in the same cells
    "vm_fp64": lambda: plastic_cube(64),
    "vm_fp32": lambda: plastic_cube(32),
    "vmmix_fp64": lambda: two_material(64, (0, 0), (1500.0, 0.0)),
    # per-cell PSD-projected Hessian on an indefinite (compressed) state
    "psd_fp64": lambda: compressed_cube(64),
    "psd_fp32": lambda: compressed_cube(32),
    "psdI_fp32": lambda: compressing_cube(32),
    "psdI_fp64": lambda: compressing_cube(64),
}


def _fp32_scene(sc):
    # cfg1(prestrain, precision=32) builds fp64 arrays for F; quantise every input to the precision
    dt_ = sc.dtype
    return dataclasses.replace(sc, x=sc.x.astype(dt_), v=sc.v.astype(dt_), F=sc.F.astype(dt_), G=sc.G.astype(dt_),
                               vol=sc.vol.astype(dt_))


@pytest.fixture(scope="module", params=list(SCENES))
def pair(request):
    sc = _fp32_scene(SCENES[request.param]())
    return Pair(sc)


def test_indices_bit_exact(pair):
    sc = pair.scene
    base_o = oracle.base_cells(pair.grid, sc.x)
    base_g = pair.ctx.get_particle_cells()
    assert np.array_equal(base_o, base_g)
    blocks_o = oracle.active_blocks(pair.grid, base_o)
    assert np.array_equal(pair.ctx.get_active_blocks(), blocks_o)
    # active nodes: exactly the nodes with m_i > 0
    assert set(pair.nid.tolist()) == set(np.nonzero(pair.un.m_i > 0)[0].tolist())


def test_unload_parity(pair):
    tol = TOL[pair.scene.precision]["unload"]
    q = pair.ctx.get_quadrature()
    cid = cell_ids(pair.grid, q["ijk"])
    structural = oracle.structural_cells(pair.grid, oracle.base_cells(pair.grid, pair.scene.x))
    assert np.array_equal(np.sort(cid), structural)
    act = pair.un.m_c[cid] > 0
    assert act.sum() == np.count_nonzero(pair.un.m_c)
    assert rel_l2(q["m_c"][act], pair.un.m_c[cid][act]) <= tol
    assert rel_l2(q["v_c"][act], pair.un.v_c[cid][act]) <= tol
    assert rel_l2(q["G_c"][act], pair.un.G_c[cid][act]) <= tol
    for k in range(len(pair.scene.materials)):
        assert rel_l2(q["V_ck"][k][act], pair.un.V_ck[k][cid][act]) <= tol
        sel = pair.un.V_ck[k][cid] > 0
        if np.abs(pair.un.tau_ck[k]).max() > 0:
            assert rel_l2(q["tau_ck"][k][sel], pair.un.tau_ck[k][cid][sel]) <= tol
        assert rel_l2(q["S_ck"][k][sel], pair.S[k][cid][sel]) <= tol
    assert rel_l2(pair.m, pair.un.m_i[pair.nid]) <= tol
    assert rel_l2(pair.vn, pair.un.v_i[pair.nid]) <= tol
    fixed = (pair.prob.freed[pair.nid] == 0)
    assert np.array_equal(pair.free.astype(bool), ~fixed)


def _probe(pair):
    rng = np.random.default_rng(5)
    v = pair.v0 + 0.01 * rng.normal(size=pair.v0.shape) * (pair.un.m_i > 0)[:, None]
    if pair.scene.precision == 32:
        v = v.astype(np.float32).astype(np.float64)
    u = np.random.default_rng(4).normal(size=pair.v0.shape) * (pair.un.m_i > 0)[:, None]
    if pair.scene.precision == 32:
        u = u.astype(np.float32).astype(np.float64)
    return v, u


def _at(pair, v):
    """The oracle problem the GPU evaluates at v: with fixed-point plasticity the gradient and the full
    linearisation re-project the bases at v; otherwise the resample's bases.  The Hessian mode
    (exact / PSD-projected) follows the scene's solver, and the GPU context is set to the same."""
    psd = bool(getattr(pair.scene.solver, "psd", False))
    pair.ctx.set_psd_projection(psd)
    if any(getattr(m, "yield_stress", 0.0) > 0 for m in pair.scene.materials):
        return pair.prob.with_bases(pair.prob.plastic_update(v)[0]).with_psd(psd)
    return pair.prob.with_psd(psd)


def test_energy_gradient_parity(pair):
    tol = TOL[pair.scene.precision]["grad"]
    v, _ = _probe(pair)
    po = _at(pair, v)
    g_o = po.gradient(v)
    g_g, phi_g = pair.ctx.gradient(pair.to_gpu(v))
    assert rel_l2(g_g, g_o[pair.nid]) <= tol
    phi_o = po.energy(v)
    assert abs(phi_g - phi_o) <= tol * abs(phi_o)
    assert abs(pair.ctx.energy(pair.to_gpu(v)) - phi_o) <= tol * abs(phi_o)


def test_hvp_and_diag_parity(pair):
    tol = TOL[pair.scene.precision]["hvp"]
    v, u = _probe(pair)
    po = _at(pair, v)
    pair.ctx.linearize(pair.to_gpu(v))
    h_o = po.hvp(v, u)
    h_g = pair.ctx.hvp(pair.to_gpu(u))
    assert rel_l2(h_g, h_o[pair.nid]) <= tol
    # elastic part alone (the mass term is exact and could hide tangent errors).  The GPU returns Hu
    # rounded to its precision, so the part recovered by subtracting m u carries that rounding, at most
    # a few eps |m u| (DESIGN.md §9 reading r2-a): bar = tol |el| + 4 eps |m u|
    m = pair.un.m_i[:, None]
    el_o = (h_o - m * u)[pair.nid]
    el_g = h_g - pair.m[:, None] * pair.to_gpu(u)
    eps = 2.0 ** -24 if pair.scene.precision == 32 else 2.0 ** -53
    mu_ = np.linalg.norm((m * u)[pair.nid])
    assert np.linalg.norm(el_g - el_o) <= tol * np.linalg.norm(el_o) + 4 * eps * mu_
    d_o = po.diag(v)
    assert rel_l2(pair.ctx.get_diag(), d_o[pair.nid]) <= tol


def test_full_step_parity(pair):
    """One implicit step with the oracle's Newton / PCG / line-search counts replayed."""
    sc = pair.scene
    tol = TOL[sc.precision]["step"]
    st_o = pair.prob.newton(pair.v0, sc.solver)[1]
    v_o, _ = pair.prob.newton(pair.v0, sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    ctx = pair.ctx
    ctx.set_velocity(pair.to_gpu(pair.v0))
    st_g = ctx.newton_step(sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    assert st_g["newton_iters"] == st_o["newton_iters"]
    assert st_g["cg_iters"] == st_o["cg_iters"]
    v_g = ctx.get_velocity()
    assert rel_l2(v_g, v_o[pair.nid]) <= tol
    ctx.transfer_to_particles(sc.dt)
    x_g, vp_g, F_g, G_g = ctx.get_particles()
    x_o, vp_o, F_o, G_o = oracle.g2p(pair.grid, sc.dt, pair.un.m_c, v_o, sc.x, sc.v, sc.F, sc.G, mat=sc.mat,
                                     materials=sc.materials)
    assert rel_l2(x_g, x_o) <= tol
    assert rel_l2(vp_g, vp_o) <= tol
    assert rel_l2(F_g, F_o) <= tol
    assert rel_l2(G_g, G_o) <= tol


def test_adaptive_solve_converges(pair):
    """Without replay the GPU solver reaches the oracle's tolerances on its own."""
    sc = pair.scene
    ctx = pair.ctx
    ctx.set_particles(sc.x, sc.v, sc.F, sc.G, sc.vol, sc.mat)  # the step test advected them
    ctx.resample(sc.dt)
    st = ctx.newton_step(sc.solver)
    assert st["converged"] == 1
    v_o, st_o = pair.prob.newton(pair.v0, sc.solver)
    # two independent adaptive solves (own counts), each stopped at ||g|| <= eps_N ||g_0||: they agree to
    # the solver tolerance, not to rounding (DESIGN.md §9 reading r2-c)
    assert rel_l2(ctx.get_velocity(), v_o[pair.nid]) <= (1e-7 if sc.precision == 64 else 1e-3)
    # the reported Phi is the energy at the returned velocity (reused from the last linearisation / accepted
    # line-search trial, not recomputed): it matches a fresh energy evaluation there
    e_now = ctx.energy(ctx.get_velocity())
    assert abs(st["energy"] - e_now) <= (1e-12 if sc.precision == 64 else 1e-6) * abs(e_now)
