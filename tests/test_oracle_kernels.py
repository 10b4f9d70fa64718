"""Oracle pins, part 1: Q1 kernels (C1), eigen, StVK-Hencky stress/energy (C2), stretch (C5).

Every check ties the oracle to something other than itself: worked examples of the
paper/SPEC (tests/golden), closed forms, library routines on special cases, finite
differences, invariants (isotropy, objectivity).  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def rand_rot(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))[None, :]
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


# ---------------------------------------------------------------- C1 Q1 weights
def test_q1_partition_first_moment(orc):
    """P:722-727 (App. A): sum_c w_cp = 1 and sum_c w_cp x_c = x for all x."""
    rng = np.random.default_rng(0)
    g = orc.Grid((8, 8, 8), 0.125)
    for _ in range(200):
        x = rng.uniform(0.2, 0.8, size=3)
        b = orc.base_cells(g, x[None])[0]
        f = x / g.dx - 0.5 - b
        assert np.all(f >= 0) and np.all(f < 1)
        w = orc.q1_weights(f)
        assert abs(w.sum() - 1) < 1e-14
        xc = np.array([[(b[0] + ((o >> 2) & 1) + 0.5) * g.dx, (b[1] + ((o >> 1) & 1) + 0.5) * g.dx,
                        (b[2] + (o & 1) + 0.5) * g.dx] for o in range(8)])
        assert np.allclose((w[:, None] * xc).sum(0), x, atol=1e-14)
        assert np.all(w >= 0)


def test_q1_interpolation_and_corner(orc):
    """x at a centre -> weight 1 there; S:38 (tensor product): x at the common corner of 8
    centres -> 1/8 each; 1D midpoint -> 1/2."""
    g = orc.Grid((8, 8, 8), 0.125)
    xc = (np.array([3, 4, 5]) + 0.5) * g.dx
    b = orc.base_cells(g, xc[None])[0]
    assert list(b) == [3, 4, 5]
    w = orc.q1_weights(xc / g.dx - 0.5 - b)
    assert w[0] == 1.0 and np.all(w[1:] == 0)
    corner = np.array([4, 4, 4]) * g.dx  # a node = common corner of 8 centres
    b = orc.base_cells(g, corner[None])[0]
    w = orc.q1_weights(corner / g.dx - 0.5 - b)
    assert np.allclose(w, 1 / 8, atol=0)
    # tensor product: weight factorises into 1D tents
    f = np.array([0.3, 0.6, 0.9])
    w = orc.q1_weights(f)
    one = lambda fa, o: fa if o else 1 - fa
    for o in range(8):
        assert w[o] == pytest.approx(one(f[0], (o >> 2) & 1) * one(f[1], (o >> 1) & 1) * one(f[2], o & 1), abs=1e-16)


def test_base_cell_bruteforce(orc):
    """C1 base cell = the centre with largest coordinates <= x per axis (brute force over centres)."""
    rng = np.random.default_rng(1)
    g = orc.Grid((16, 16, 16), 1 / 16)
    x = rng.uniform(0.05, 0.95, size=(500, 3))
    b = orc.base_cells(g, x)
    cen = (np.arange(16) + 0.5) / 16
    for a in range(3):
        bf = np.array([np.max(np.nonzero(cen <= xx)[0]) for xx in x[:, a]])
        assert np.array_equal(b[:, a], bf)


# ---------------------------------------------------------------- eigen
def test_sym_eig3_vs_library(orc):
    """Special case reducing to a library routine: eigenvalues match numpy.linalg.eigvalsh and
    A = Q diag(w) Q^T with orthonormal Q, including repeated eigenvalues."""
    rng = np.random.default_rng(2)
    mats = [rng.normal(size=(3, 3)) for _ in range(100)]
    mats = [m + m.T for m in mats]
    mats += [np.diag([1.0, 1.0, 2.0]), np.eye(3) * 3.0, np.zeros((3, 3))]
    R = rand_rot(rng)
    mats.append(R @ np.diag([0.5, 0.5, -1.0]) @ R.T)
    for A in mats:
        w, Q = orc.sym_eig3(A)
        assert np.allclose(np.sort(w), np.linalg.eigvalsh(A), atol=1e-13 * (1 + np.abs(A).max()))
        assert np.allclose(Q @ Q.T, np.eye(3), atol=1e-13)
        assert np.allclose(Q @ np.diag(w) @ Q.T, A, atol=1e-13 * (1 + np.abs(A).max()))


# ---------------------------------------------------------------- C2 Hencky
def test_hencky_worked_examples(orc):
    ex = GOLD["hencky_stress_diag"]
    tau = orc.hencky_tau(np.diag(ex["F"]), ex["mu"], ex["lam"])
    assert np.allclose(np.diag(tau), ex["expected_tau_diag"], atol=1e-14)
    assert np.allclose(tau - np.diag(np.diag(tau)), 0, atol=1e-15)
    assert np.all(orc.hencky_tau(np.eye(3), 3.0, 7.0) == GOLD["hencky_rest"]["expected"])


def test_hencky_closed_form_diagonal(orc):
    """Eq. hencky-energy / hencky-taui on diagonal F = diag(sigma): closed forms."""
    for sig in ([1.2, 0.9, 1.05], [2.0, 0.5, 1.0], [0.7, 0.7, 1.3]):
        mu, lam = 3.0, 5.0
        e = np.log(sig)
        psi = mu * (e ** 2).sum() + 0.5 * lam * e.sum() ** 2
        assert orc.hencky_psi(np.diag(sig), mu, lam) == pytest.approx(psi, rel=1e-13)
        tau = orc.hencky_tau(np.diag(sig), mu, lam)
        assert np.allclose(np.diag(tau), 2 * mu * e + lam * e.sum(), rtol=1e-13, atol=1e-14)


def test_hencky_tau_is_dpsi_dF_FT(orc):
    """tau = P F^T with P = d psi / dF — central finite differences of psi."""
    rng = np.random.default_rng(3)
    mu, lam = 2.0, 3.0
    for _ in range(10):
        F = np.eye(3) + 0.3 * rng.normal(size=(3, 3))
        if np.linalg.det(F) < 0.2:
            continue
        h = 1e-6
        P = np.zeros((3, 3))
        for a in range(3):
            for b in range(3):
                Fp, Fm = F.copy(), F.copy()
                Fp[a, b] += h
                Fm[a, b] -= h
                P[a, b] = (orc.hencky_psi(Fp, mu, lam) - orc.hencky_psi(Fm, mu, lam)) / (2 * h)
        tau = orc.hencky_tau(F, mu, lam)
        assert np.allclose(P @ F.T, tau, rtol=1e-7, atol=1e-7)
        assert np.allclose(tau, tau.T, atol=1e-13)


def test_hencky_isotropy(orc):
    """Eq. isotropy: psi(Q1 F Q2) = psi(F); tau(F Q) = tau(F); tau(Q F) = Q tau Q^T."""
    rng = np.random.default_rng(4)
    for _ in range(20):
        F = np.eye(3) + 0.2 * rng.normal(size=(3, 3))
        Q1, Q2 = rand_rot(rng), rand_rot(rng)
        assert orc.hencky_psi(Q1 @ F @ Q2, 1.5, 2.5) == pytest.approx(orc.hencky_psi(F, 1.5, 2.5), rel=1e-11)
        t = orc.hencky_tau(F, 1.5, 2.5)
        assert np.allclose(orc.hencky_tau(F @ Q2, 1.5, 2.5), t, atol=1e-12)
        assert np.allclose(orc.hencky_tau(Q1 @ F, 1.5, 2.5), Q1 @ t @ Q1.T, atol=1e-12)
    with pytest.raises(ValueError):
        orc.hencky_tau(np.diag([1.0, 1.0, -1.0]), 1.0, 1.0)


# ---------------------------------------------------------------- C5 stretch
def test_stretch_worked_examples(orc):
    ex = GOLD["hencky_inversion_spherical"]
    S = orc.stretch(np.diag(ex["tau_diag"]), ex["mu"], ex["lam"])
    assert np.allclose(S, ex["expected_sigma"] * np.eye(3), atol=1e-14)
    assert np.allclose(orc.stretch(np.zeros((3, 3)), 2.0, 3.0), np.eye(3), atol=0)


def test_stretch_round_trip_and_objectivity(orc):
    """Eq. rotfree-def: P(S) S^T = tau — round trip tau(S(tau)) = tau; S SPD; and
    objectivity S(Q tau Q^T) = Q S(tau) Q^T; repeated eigenvalues."""
    rng = np.random.default_rng(5)
    mu, lam = 3846.15, 5769.23
    for _ in range(50):
        R = rand_rot(rng)
        sig = rng.uniform(0.5, 2.0, size=3)
        S_true = R @ np.diag(sig) @ R.T
        tau = orc.hencky_tau(S_true, mu, lam)
        S = orc.stretch(tau, mu, lam)
        assert np.allclose(S, S_true, rtol=1e-10, atol=1e-10)
        assert np.allclose(orc.hencky_tau(S, mu, lam), tau, rtol=1e-10, atol=1e-10 * np.abs(tau).max())
        Q = rand_rot(rng)
        assert np.allclose(orc.stretch(Q @ tau @ Q.T, mu, lam), Q @ S @ Q.T, atol=1e-10)
    # repeated eigenvalues: any basis of the eigenspace gives the same S
    R = rand_rot(rng)
    tau = R @ np.diag([100.0, 100.0, -50.0]) @ R.T
    S = orc.stretch(tau, mu, lam)
    e = (np.array([100.0, 100.0, -50.0]) - lam * 150.0 / (2 * mu + 3 * lam)) / (2 * mu)
    assert np.allclose(S, R @ np.diag(np.exp(e)) @ R.T, atol=1e-13)
