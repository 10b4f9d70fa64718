"""Edge cases of the C-ABI path on the GPU: empty input, a single particle, particles exactly on
cell-centre planes (zero-weight stencil cells, amb-10), the error classes of SURVEY §8(b) (out of
domain, inverted element, call order, invalid arguments), the grid-size limit, and a ragged scene
whose tiles are partially filled and whose particle count is not a multiple of any block size."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2602_07853_b200 import mpl, scenes

from ._parity import node_ids, rel_l2

pytestmark = pytest.mark.gpu


def one_particle_scene(x, precision=64):
    x = np.asarray(x, np.float64).reshape(1, 3)
    n = 16
    return scenes._assemble("one", precision, n, 1e-3, [scenes.Material(1e4, 0.3, 1000.0)], x,
                            np.array([[1.0, 0.0, 0.0]]), np.eye(3).reshape(1, 9), np.zeros((1, 9)),
                            np.zeros(1, np.int32), 8, [], scenes.SolverCfg(eps_cg=1e-10, eps_newton=1e-10), 1)


def test_empty_input():
    sc = one_particle_scene([0.5, 0.5, 0.5])
    ctx = mpl.Context(sc.n, sc.dx, 64, 0)
    ctx.set_materials(sc.materials)
    e3, e9 = np.zeros((0, 3)), np.zeros((0, 9))
    ctx.set_particles(e3, e3, e9, e9, np.zeros(0), np.zeros(0, np.int32))
    c = ctx.resample(sc.dt)
    assert (c.n_cells, c.n_nodes, c.n_blocks) == (0, 0, 0)
    st = ctx.newton_step(sc.solver)
    assert st["cg_total"] == 0
    ctx.transfer_to_particles(sc.dt)
    x, v, F, G = ctx.get_particles()
    assert x.shape == (0, 3)
    st = ctx.step(sc.dt, sc.solver)
    assert st["n_cells"] == 0
    ctx.close()


def test_single_particle_at_centre():
    """one particle at a cell centre, v_p = (1,0,0), G_p = 0 -> 8 nodes carry m_p/8 and v_p."""
    sc = one_particle_scene([(7 + 0.5) / 16, (8 + 0.5) / 16, (9 + 0.5) / 16])
    ctx = mpl.from_scene(sc, 0)
    c = ctx.resample(sc.dt)
    ijk, m, vn, fr = ctx.get_nodes()
    mp = sc.materials[0].rho * sc.vol[0]
    assert c.n_nodes == 8
    assert np.allclose(m, mp / 8, rtol=1e-14)
    assert np.allclose(vn, [[1.0, 0.0, 0.0]] * 8, atol=1e-14)
    assert sorted(map(tuple, ijk.tolist())) == sorted((7 + a, 8 + b, 9 + d) for a in (0, 1) for b in (0, 1) for d in (0, 1))
    # F = I, uniform v: the Newton start v-hat = v + dt g (amb-4) is already the minimiser, g is rounding
    # noise (~1e-23) and the relative Newton test need not fire (the oracle runs to newton_max as well);
    # the velocities must stay at v-hat
    st = ctx.newton_step(sc.solver)
    assert st["newton_iters"] >= 1
    vhat = np.array([1.0, 0.0, 0.0]) + sc.dt * np.asarray(sc.gravity)
    assert np.allclose(ctx.get_velocity(), [vhat] * 8, atol=1e-12)
    ctx.close()


def test_particles_on_centre_planes_match_oracle():
    """Lattice particles on cell-centre planes: f = 0 exactly on some axes, so stencil cells with
    zero weight (m_c = 0) stay structural (amb-10); unload, gradient, HVP and a full step still match."""
    n = 16
    cells = scenes.cells_box([4, 4, 4], [10, 9, 11])
    x = (cells + 0.5) / n  # exactly at centres: base cell = the cell, weight 1 on it, 0 on 7 others
    x = np.concatenate([x, (cells + np.array([0.5, 0.75, 0.5])) / n])  # and half-way in y only
    rng = np.random.default_rng(3)
    v = 0.1 * rng.normal(size=x.shape)
    sc = scenes._assemble("planes", 64, n, 1e-3, [scenes.Material(1e5, 0.3, 1000.0)], x, v,
                          scenes._prestrain(x.shape[0], 3), np.zeros((x.shape[0], 9)),
                          np.zeros(x.shape[0], np.int32), 1, [],
                          scenes.SolverCfg(eps_cg=1e-10, eps_newton=1e-10), 1)
    grid = oracle.Grid(sc.n, sc.dx, sc.origin)
    un, S, prob, v0 = oracle.prepare(sc, grid)
    assert np.any(un.m_c == 0) and np.any(un.m_c > 0)
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    ijk, m, vn, fr = ctx.get_nodes()
    nid = node_ids(grid, ijk)
    assert set(nid.tolist()) == set(np.nonzero(un.m_i > 0)[0].tolist())
    assert rel_l2(m, un.m_i[nid]) <= 1e-12
    g, _ = ctx.gradient(np.ascontiguousarray(v0[nid]))
    assert rel_l2(g, prob.gradient(v0)[nid]) <= 1e-10
    st_o = prob.newton(v0, sc.solver)[1]
    v_o, _ = prob.newton(v0, sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    ctx.set_velocity(np.ascontiguousarray(v0[nid]))
    ctx.newton_step(sc.solver, st_o["newton_iters"], st_o["cg_iters"], st_o["ls_iters"])
    assert rel_l2(ctx.get_velocity(), v_o[nid]) <= 1e-8
    ctx.close()


def test_ragged_scene_full_step():
    """A random blob: tiles partly filled, counts not multiples of 4 / 32 / 64; full step vs oracle."""
    n = 16
    rng = np.random.default_rng(11)
    x = 0.25 + 0.45 * rng.random((1237, 3))
    v = 0.2 * rng.normal(size=x.shape)
    sc = scenes._assemble("ragged", 64, n, 1e-3, [scenes.Material(3e4, 0.25, 800.0)], x, v,
                          scenes._prestrain(x.shape[0], 3), 0.3 * rng.normal(size=(x.shape[0], 9)),
                          np.zeros(x.shape[0], np.int32), 3, [],
                          scenes.SolverCfg(eps_cg=1e-10, eps_newton=1e-10), 1)
    r = oracle.step(sc)
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    st = ctx.newton_step(sc.solver, r.stats["newton_iters"], r.stats["cg_iters"], r.stats["ls_iters"])
    assert st["cg_iters"] == r.stats["cg_iters"]
    ctx.transfer_to_particles(sc.dt)
    xg, vg, Fg, Gg = ctx.get_particles()
    for a, b in ((xg, r.particles[0]), (vg, r.particles[1]), (Fg, r.particles[2])):
        assert rel_l2(a, b) <= 1e-8
    ctx.close()


def test_error_classes():
    sc = scenes.cfg1()
    # out of domain: a base cell above N-2 (the stencil would leave the grid)
    x = sc.x.copy()
    x[17, 2] = 0.999
    ctx = mpl.from_scene(dataclasses.replace(sc, x=x), 0)
    with pytest.raises(mpl.MplError) as e:
        ctx.resample(sc.dt)
    assert e.value.code == 3 and "17" in str(e.value)
    ctx.close()
    # inverted element: det F_p <= 0
    F = sc.F.copy()
    F[5] = np.diag([1.0, 1.0, -1.0]).ravel()
    ctx = mpl.from_scene(dataclasses.replace(sc, F=F), 0)
    with pytest.raises(mpl.MplError) as e:
        ctx.resample(sc.dt)
    assert e.value.code == 4 and "5" in str(e.value)
    # the failed resample left the state unresampled: call-order error, not a crash
    with pytest.raises(mpl.MplError) as e:
        ctx.hvp(np.zeros((1, 3)))
    assert e.value.code == 2
    ctx.close()
    # call order on a fresh context
    ctx = mpl.from_scene(sc, 0)
    with pytest.raises(mpl.MplError) as e:
        ctx.linearize(np.zeros((1, 3)))
    assert e.value.code == 2
    ctx.resample(sc.dt)
    with pytest.raises(mpl.MplError) as e:  # hvp before linearize
        ctx.hvp(np.zeros((ctx.counts.n_nodes, 3)))
    assert e.value.code == 2
    ctx.close()
    # invalid material / precision / grid
    ctx = mpl.Context(sc.n, sc.dx, 64, 0)
    with pytest.raises(mpl.MplError):
        ctx.set_materials([scenes.Material(1e4, 0.6, 1000.0)])  # lam < -2mu/3
    with pytest.raises(mpl.MplError):
        ctx.set_materials([scenes.Material(1e4, 0.3, 1000.0, 7)])  # unknown law
    ctx.close()
    with pytest.raises(mpl.MplError):
        mpl.Context(sc.n, sc.dx, 16, 0)
    with pytest.raises(mpl.MplError):
        mpl.Context((1023, 8, 8), 1.0 / 1023, 32, 0)


def test_largest_grid_extent_accepted():
    """The grid limit is 1022 cells per axis (10-bit packed base cells); a thin 1022 x 8 x 8 slab runs."""
    n0 = 1022
    dx = 1.0 / 1024
    cells = scenes.cells_box([1000, 2, 2], [1010, 6, 6])
    x = (cells + 0.5) * dx
    v = 0.1 * np.random.default_rng(2).normal(size=x.shape)
    sc = scenes._assemble("long", 32, n0, 1e-3, [scenes.Material(1e4, 0.3, 1000.0)], x,
                          v, scenes._prestrain(x.shape[0], 3),
                          np.zeros((x.shape[0], 9)), np.zeros(x.shape[0], np.int32), 1, [],
                          scenes.SolverCfg(), 1)
    sc = dataclasses.replace(sc, n=(n0, 8, 8), dx=dx)
    ctx = mpl.from_scene(sc, 0)
    st = ctx.step(sc.dt, sc.solver)
    assert st["converged"] == 1
    ctx.close()


def test_pipelined_io_matches_synchronous():
    """mpl_stage_particles / mpl_get_particles_async (copy streams) give the same three steps as
    mpl_set_particles / mpl_step / mpl_get_particles; the host input arrays are re-staged every step."""
    sc = scenes.cfg1(prestrain=True)
    host = [np.ascontiguousarray(a, np.float64) for a in (sc.x, sc.v, sc.F, sc.G, sc.vol)]
    mat = np.ascontiguousarray(sc.mat, np.int32)
    a = mpl.from_scene(sc, 0)
    ref = []
    for _ in range(3):
        a.set_particles(*host, mat)
        a.step(sc.dt, sc.solver)
        ref.append(a.get_particles())
    a.close()
    b = mpl.from_scene(sc, 0)
    n = sc.n_particles
    outs = [[np.zeros((n, w)) for w in (3, 3, 9, 9)] for _ in range(3)]
    b.stage_particles(*host, mat)
    with pytest.raises(mpl.MplError):  # one staged set at a time
        b.stage_particles(*host, mat)
    for i in range(3):
        b.resample(sc.dt)
        if i < 2:
            b.stage_particles(*host, mat)
        b.newton_step(sc.solver)
        b.transfer_to_particles(sc.dt)
        b.get_particles_async(*outs[i])
    b.stage_wait()
    b.close()
    # face-node float atomics make the sums order-dependent: equal to rounding, not bitwise
    for i in range(3):
        for got, want in zip(outs[i], ref[i]):
            assert rel_l2(got, want) <= 1e-12


def _affine_scene():
    """A pre-strained 16^3 block of a 32^3 grid with the cfg2 smooth field (v, G_p = grad v non-zero),
    particles given in a shuffled order so the resample's sort moves every array."""
    n = 32
    cells = scenes.cells_box([8, 8, 8], [24, 24, 24])
    x = scenes.stratified(cells, n, 2, seed=0)
    perm = np.random.default_rng(7).permutation(x.shape[0])
    x = x[perm]
    v, G = scenes.eval_smooth_field(x, scenes.smooth_field(2))
    return scenes._assemble("affine", 64, n, 2e-3, [scenes.Material(1e5, 0.4, 1000.0)], x, v,
                            scenes._prestrain(x.shape[0], 3), G, np.zeros(x.shape[0], np.int32), 8, [],
                            scenes.SolverCfg(eps_cg=1e-10, eps_newton=1e-10), 1)


def test_resample_twice_equals_once():
    """mpl_resample sorts x / F; v / G are brought into the same order before anything else
    reads them, so resample -> resample -> step equals resample -> step, and mpl_get_particles right
    after a resample returns the input state."""
    sc = _affine_scene()
    a = mpl.from_scene(sc, 0)
    a.resample(sc.dt)
    x, v, F, G = a.get_particles()  # between resample and transfer: input order, v / G unscrambled
    assert np.array_equal(x, sc.x) and np.array_equal(v, sc.v) and np.array_equal(F, sc.F) and np.array_equal(G, sc.G)
    a.resample(sc.dt)  # the recovery path of the header (mpl_resample again)
    sa = a.newton_step(sc.solver)
    va = a.get_velocity()
    a.transfer_to_particles(sc.dt)
    pa = a.get_particles()
    a.close()
    b = mpl.from_scene(sc, 0)
    b.resample(sc.dt)
    sb = b.newton_step(sc.solver, sa["newton_iters"], sa["cg_iters"], sa["ls_iters"])
    vb = b.get_velocity()
    b.transfer_to_particles(sc.dt)
    pb = b.get_particles()
    b.close()
    assert sb["cg_iters"] == sa["cg_iters"]
    assert rel_l2(va, vb) <= 1e-12
    for got, want in zip(pa, pb):
        assert rel_l2(got, want) <= 1e-12


def test_particle_cells_only_between_resample_and_transfer():
    """mpl_get_particle_cells reports the last resample's binning; after the transfer moved the particles it
    is a call-order error (it used to return the pre-advection cells)."""
    sc = _affine_scene()
    ctx = mpl.from_scene(sc, 0)
    ctx.resample(sc.dt)
    grid = oracle.Grid(sc.n, sc.dx, sc.origin)
    assert np.array_equal(ctx.get_particle_cells(), oracle.base_cells(grid, sc.x))
    ctx.newton_step(sc.solver)
    ctx.transfer_to_particles(sc.dt)
    with pytest.raises(mpl.MplError) as e:
        ctx.get_particle_cells()
    assert e.value.code == 2  # MPL_ERR_STATE
    ctx.close()
