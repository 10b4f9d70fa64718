"""Oracle pins for the split Neo-Hookean law (PAPER §4.3.2, App. C
P:1297-1348): worked example S:286, closed forms (rest, pure dilation, isochoric shear), stress as
the derivative of the energy by central finite differences (tau = dPsi/dF F^T), isotropy, the
Cardano root against a brute-force polynomial solve, and stress -> stretch round trips that exercise
both Cardano branches.  The gradient / HVP / Newton pins with this law are in
tests/test_oracle_solver.py (parametrised over the material kind)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def rand_rot(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    return q if np.linalg.det(q) > 0 else -q


def test_worked_example_s286(orc):
    ex = GOLD["split_nh_stress_3d"]
    F = np.diag(ex["F"])
    tau = orc.nh_tau(F, ex["mu"], ex["kappa"])
    assert np.allclose(np.diag(tau), ex["expected_tau_diag"], rtol=0, atol=1e-12)
    assert abs(np.trace(tau) / 3 - ex["expected_alpha"]) < 1e-12
    S, br = orc.nh_stretch(tau, ex["mu"], ex["kappa"])
    assert np.allclose(S, np.diag(ex["expected_sigma"]), atol=1e-10)
    # the cubic of the example: m^3 - 3 m - 2 = 0 with admissible root m = 2 (delta = (2,-1,-1))
    m, _ = orc.nh_cardano(-3.0, 2.0 - ex["expected_J"] ** 2, -1.0)
    assert abs(m - ex["expected_m"]) < 1e-7


def test_hand_derivation_matches(orc):
    ex = GOLD["split_nh_stress_2d_hand"]
    # tau = mu J^{-2/3} dev(b) + kappa/2 (J^2-1) I for F = diag(2,1,1), mu = kappa = 1
    tau = orc.nh_tau(np.diag([2.0, 1.0, 1.0]), 1.0, 1.0)
    expect = ex["J_pow"] * np.array(ex["dev_b"]) + 1.5
    assert np.allclose(np.diag(tau), expect, atol=1e-13)


def test_rest_dilation_and_isochoric_closed_forms(orc):
    mu, kappa = 3.7, 11.0
    assert np.allclose(orc.nh_tau(np.eye(3), mu, kappa), 0, atol=1e-15)
    assert abs(orc.nh_psi(np.eye(3), mu, kappa)) < 1e-15
    for g in (0.8, 1.0, 1.3):  # pure dilation: tau = alpha(J) I, alpha = kappa/2 (J^2-1), J = g^3
        J = g ** 3
        tau = orc.nh_tau(g * np.eye(3), mu, kappa)
        assert np.allclose(tau, 0.5 * kappa * (J * J - 1) * np.eye(3), atol=1e-12)
        assert abs(orc.nh_psi(g * np.eye(3), mu, kappa) - 0.25 * kappa * (J * J - 1 - 2 * np.log(J))) < 1e-12
    a = 1.4  # isochoric (J = 1): tau = mu dev(b)
    F = np.diag([a, 1 / a, 1.0])
    b = F @ F.T
    assert np.allclose(orc.nh_tau(F, mu, kappa), mu * (b - np.trace(b) / 3 * np.eye(3)), atol=1e-12)


def test_tau_is_energy_derivative_fd(orc):
    rng = np.random.default_rng(7)
    mu, kappa = 2.0, 5.0
    for _ in range(10):
        F = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
        if np.linalg.det(F) <= 0.2:
            continue
        P = np.zeros((3, 3))
        h = 1e-6
        for i in range(3):
            for j in range(3):
                Fp, Fm = F.copy(), F.copy()
                Fp[i, j] += h
                Fm[i, j] -= h
                P[i, j] = (orc.nh_psi(Fp, mu, kappa) - orc.nh_psi(Fm, mu, kappa)) / (2 * h)
        tau = orc.nh_tau(F, mu, kappa)
        assert np.linalg.norm(P @ F.T - tau) <= 1e-7 * max(1.0, np.linalg.norm(tau))
        assert np.allclose(tau, tau.T, atol=1e-12)


def test_isotropy(orc):
    rng = np.random.default_rng(8)
    mu, kappa = 1.5, 4.0
    for _ in range(5):
        F = np.eye(3) + 0.2 * rng.normal(size=(3, 3))
        Q = rand_rot(rng)
        t = orc.nh_tau(F, mu, kappa)
        assert np.allclose(orc.nh_tau(F @ Q, mu, kappa), t, atol=1e-12)          # tau(FQ) = tau(F)
        assert np.allclose(orc.nh_tau(Q @ F, mu, kappa), Q @ t @ Q.T, atol=1e-12)  # objectivity


def test_cardano_root_vs_polynomial_roots(orc):
    rng = np.random.default_rng(9)
    seen = set()
    for _ in range(400):
        d = rng.normal(size=3)
        d -= d.mean()                         # sum delta_i = 0
        d *= rng.choice([0.05, 0.5, 2.0])
        J = np.exp(rng.uniform(-0.5, 0.5))
        p = d[0] * d[1] + d[1] * d[2] + d[2] * d[0]
        q = d[0] * d[1] * d[2] - J * J
        m, br = orc.nh_cardano(p, q, d.min())
        seen.add(br)
        roots = np.roots([1.0, 0.0, p, q])
        real = roots[np.abs(roots.imag) < 1e-6].real
        adm = real[real > -d.min()]
        assert len(adm) >= 1
        # np.roots and the closed form both lose ~sqrt(eps) near a double root: compare loosely and
        # pin the closed form by its residual on the cubic (Eq. m-3D)
        assert abs(m - adm.max()) <= 1e-6 * max(1.0, abs(m))
        scale = abs(m) ** 3 + abs(p * m) + abs(q)
        assert abs(m ** 3 + p * m + q) <= 1e-9 * scale  # closed form; orc_nh_stretch polishes it
        assert np.all(m + d > 0)
    assert seen == {1, 3}, "both Cardano branches must be exercised"


def test_stretch_round_trip_both_branches(orc):
    rng = np.random.default_rng(10)
    branches = {1: 0, 3: 0}
    for _ in range(400):
        sig = rng.uniform(0.5, 2.0, size=3)
        if rng.random() < 0.3:
            sig[1] = sig[2]  # repeated stretches
        Q = rand_rot(rng)
        S = Q @ np.diag(sig) @ Q.T
        mu, kappa = rng.uniform(0.5, 5.0), rng.uniform(0.5, 20.0)
        tau = orc.nh_tau(S, mu, kappa)
        S2, br = orc.nh_stretch(tau, mu, kappa)
        branches[br] += 1
        assert np.linalg.norm(S2 - S) <= 1e-10 * np.linalg.norm(S)
    assert branches[1] > 0 and branches[3] > 0
