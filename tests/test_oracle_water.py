"""Oracle pins for the J-based water slots (PAPER §4.5).

psi(J) = kappa/2 (J - 1)^2, pi(J) = J psi'(J) = kappa J (J - 1), tau = pi I; unload of the pressure
moment; J_base = (1 + sqrt(1 + 4 pi / kappa)) / 2; J_p^{n+1} = (1 + dt tr G_p) J_p^n.  Pins: the
worked values of the SPEC (kappa = 2, J = 2 -> pi = 4 -> J_base = 2; pi = 0 -> 1;
pi = -kappa/4 -> 1/2), tau = (d psi / dF) F^T by central differences, round trips, the unload of a
uniform-J block (pi_c = pi(J), J_base = J), and the trace-form J update under an exact affine dilation.
The solver pins of test_oracle_solver.py (FD gradient / HVP, symmetry, diagonal, one-point
stiffness kappa tr(eps) I, patch test, rigid rotation, brute-force Newton) run for water (kind 2)
and a Hencky + water mixture."""
import dataclasses

import numpy as np
import pytest

from paper_2602_07853_b200 import scenes


def test_spec_worked_values(orc):
    assert orc.water_pi(1.0, 2.0) == 0.0  # rest state
    assert orc.water_pi(2.0, 2.0) == pytest.approx(4.0, abs=1e-15)  # kappa=2, J=2 -> pi = 4
    assert orc.water_jbase(4.0, 2.0) == pytest.approx(2.0, abs=1e-15)  # (1 + sqrt(9)) / 2
    assert orc.water_jbase(0.0, 2.0) == 1.0
    assert orc.water_jbase(-0.5, 2.0) == pytest.approx(0.5, abs=1e-15)  # pi = -kappa/4: branch minimum
    assert orc.water_jbase(-0.6, 2.0) == 0.5  # radicand clamped at 0
    assert orc.water_psi_J(3.0, 5.0) == pytest.approx(10.0)  # kappa/2 (J-1)^2


@pytest.mark.parametrize("kappa", [2.0, 3.7e6])
def test_round_trip_positive_branch(orc, kappa):
    for J in np.linspace(0.51, 3.0, 40):
        assert orc.water_jbase(orc.water_pi(J, kappa), kappa) == pytest.approx(J, rel=1e-12)


def test_tau_is_psi_derivative(orc):
    """tau = (d psi / dF) F^T (Kirchhoff stress of the energy) by central differences, and it
    depends on F only through det F."""
    rng = np.random.default_rng(12)
    kappa = 2.5e3
    for _ in range(6):
        F = np.eye(3) + 0.2 * rng.normal(size=(3, 3))
        if np.linalg.det(F) <= 0:
            continue
        h = 1e-7
        dpsi = np.zeros((3, 3))
        for a in range(3):
            for b in range(3):
                Fp, Fm = F.copy(), F.copy()
                Fp[a, b] += h
                Fm[a, b] -= h
                dpsi[a, b] = (orc.water_psi(Fp, kappa) - orc.water_psi(Fm, kappa)) / (2 * h)
        tau = orc.water_tau(F, kappa)
        assert np.allclose(tau, dpsi @ F.T, rtol=1e-6, atol=1e-6 * np.abs(tau).max())
        J = np.linalg.det(F)
        assert np.allclose(tau, kappa * J * (J - 1) * np.eye(3), rtol=1e-13, atol=1e-13 * kappa)
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        Q *= np.sign(np.linalg.det(Q))
        assert np.allclose(orc.water_tau(Q @ F, kappa), tau, rtol=1e-12, atol=1e-12 * kappa)  # objectivity


def test_stretch_is_isotropic_with_det_jbase(orc):
    kappa = 7.0
    for pi in (-1.5, 0.0, 0.3, 12.0):
        S = orc.water_stretch(pi * np.eye(3), kappa)
        assert np.allclose(S, S[0, 0] * np.eye(3), atol=0)
        assert np.linalg.det(S) == pytest.approx(orc.water_jbase(pi, kappa), rel=1e-14)


def water_block(J0=1.05, kappa=3e4, vel=None, n=12):
    cells = scenes.cells_box([3] * 3, [9] * 3)
    x = scenes.stratified(cells, n, 2, seed=1)
    F = np.tile((J0 ** (1 / 3) * np.eye(3)).ravel(), (x.shape[0], 1))
    v = np.zeros_like(x) if vel is None else vel(x)
    return scenes.Scene(name="w", precision=64, n=(n, n, n), dx=1 / n, dt=1e-3,
                        materials=[scenes.Material(kappa, 0.0, 1000.0, 2)], x=x, v=v, F=F,
                        G=np.zeros((x.shape[0], 9)), vol=np.full(x.shape[0], (1 / n) ** 3 / 8),
                        mat=np.zeros(x.shape[0], np.int32), dirichlet=[],
                        solver=scenes.SolverCfg(eps_cg=1e-12, eps_newton=1e-10))


def test_unload_uniform_J_reconstructs_J(orc):
    """pi_c = (1/V_c) sum_p w_cp V_p pi_p of a uniform-J block is pi(J) in every cell, and the
    reconstructed base Jacobian is J."""
    J0, kappa = 1.05, 3e4
    sc = water_block(J0, kappa)
    un, S, prob, v0 = orc.prepare(sc)
    act = un.V_ck[0] > 0
    tau = un.tau_ck[0][act]
    assert np.allclose(tau[:, [0, 4, 8]], orc.water_pi(J0, kappa), rtol=1e-12)
    assert np.allclose(tau[:, [1, 2, 3, 5, 6, 7]], 0.0, atol=1e-12 * kappa)
    detS = np.linalg.det(S[0][act].reshape(-1, 3, 3))
    assert np.allclose(detS, J0, rtol=1e-12)


def test_g2p_trace_form_under_affine_dilation(orc):
    """v_i = eps (x_i - x0) (applied on the grid): G_c = eps I exactly in every active cell (affine
    reproduction), so J_p^{n+1} = (1 + 3 dt eps) J_p^n and F_p stays J^{1/3} I."""
    eps, J0 = 0.7, 1.02
    sc = water_block(J0)
    grid = orc.Grid(sc.n, sc.dx, sc.origin)
    un = orc.unload(grid, sc.materials, sc.x, sc.v, sc.F, sc.G, sc.vol, sc.mat)
    xi = grid.node_ijk() * sc.dx
    v_i = eps * (xi - 0.5)
    x, v, F, G = orc.g2p(grid, sc.dt, un.m_c, v_i, sc.x, sc.v, sc.F, sc.G, mat=sc.mat, materials=sc.materials)
    Jn = J0 * (1 + 3 * sc.dt * eps)
    assert np.allclose(np.linalg.det(F.reshape(-1, 3, 3)), Jn, rtol=1e-13)
    assert np.allclose(F.reshape(-1, 3, 3), Jn ** (1 / 3) * np.eye(3), rtol=1e-13, atol=1e-15)
    assert np.allclose(G.reshape(-1, 3, 3), eps * np.eye(3), rtol=1e-12, atol=1e-12)


def test_pressure_pushes_outward_and_step_conserves_momentum(orc):
    """A compressed block (J = 0.95, pi = kappa J (J-1) < 0) without gravity: the implicit step moves
    it outward (net positive radial velocity; a stretched block, J = 1.1, moves inward) and the grid
    momentum stays zero (internal forces sum to zero)."""
    for J0, sign in ((0.95, 1.0), (1.1, -1.0)):
        _check_breathing(orc, J0, sign)


def _check_breathing(orc, J0, sign):
    sc = dataclasses.replace(water_block(J0), gravity=(0.0, 0.0, 0.0))
    r = orc.step(sc)
    assert r.stats["converged"] == 1
    un, prob = r.unloaded, r.problem
    act = prob.m_i > 0
    mom = (prob.m_i[act, None] * r.v_new[act]).sum(0)
    assert np.allclose(mom, 0.0, atol=1e-12 * prob.m_i.sum())
    xi = orc.Grid(sc.n, sc.dx, sc.origin).node_ijk() * sc.dx - 0.5
    radial = (r.v_new[act] * xi[act]).sum(1)
    assert sign * radial.sum() > 0
