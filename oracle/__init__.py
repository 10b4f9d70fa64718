"""CPU fp64 ORACLE for the MPM Lite hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2602_07853_b200``) never imports it, and it never imports the product path
(the shared seeded input generators live in ``paper_2602_07853_b200/scenes.py``,
which holds none of the method's arithmetic).

Thin ctypes wrapper over ``mpl_oracle.c`` (plain fp64 C, -O2 -ffp-contract=off).
All arrays are dense over a grid window (cells x-major, nodes x-major).  The
composition of the steps below follows Alg. 1: Unload (Alg. 2) →
Integrate (Alg. 3) → Load (Alg. 4).

Parity status per function: every function here is pinned by tests in
``tests/test_oracle_*.py`` (closed forms, worked examples of SPEC.md, invariants,
finite differences, brute force); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
MAXMAT = 8


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off, no fast-math, -fopenmp: results are identical at
    any OMP_NUM_THREADS, see the header of mpl_oracle.c)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB + ".tmp", _SRC, "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Grid(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("dx", C.c_double), ("origin", C.c_double * 3)]


class _Mat(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double), ("kind", C.c_int32),
                ("yield_stress", C.c_double)]


class _Box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("vel", C.c_double * 3)]


class _Problem(C.Structure):
    _fields_ = [("g", _Grid), ("nmat", C.c_int32), ("mats", _Mat * MAXMAT), ("dt", C.c_double),
                ("m_i", C.c_void_p), ("vhat", C.c_void_p), ("freed", C.c_void_p), ("m_c", C.c_void_p),
                ("V_ck", C.c_void_p), ("S_ck", C.c_void_p), ("psd", C.c_int32)]


class _SolverCfg(C.Structure):
    _fields_ = [("newton_max", C.c_int32), ("cg_max", C.c_int32), ("ls_max", C.c_int32),
                ("eps_newton", C.c_double), ("eps_cg", C.c_double), ("armijo", C.c_double),
                ("fixed_newton", C.c_int32), ("fixed_cg", C.c_void_p), ("fixed_ls", C.c_void_p),
                ("ls_slack", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("cg_total", C.c_int32), ("ls_halvings", C.c_int32),
                ("converged", C.c_int32), ("neg_curv", C.c_int32), ("grad_norm0", C.c_double),
                ("grad_norm", C.c_double), ("energy", C.c_double), ("cg_iters", C.c_int32 * 64),
                ("ls_iters", C.c_int32 * 64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        vp, i64, i32, d = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        L.orc_sym_eig3.argtypes = [vp, vp, vp]
        L.orc_base_cells.argtypes = [vp, i64, vp, vp]
        L.orc_q1_weights.argtypes = [vp, vp]
        L.orc_hencky_tau.argtypes = [vp, d, d, vp]
        L.orc_hencky_tau.restype = C.c_int
        L.orc_hencky_psi.argtypes = [vp, d, d]
        L.orc_hencky_psi.restype = d
        L.orc_p2q.argtypes = [vp, i32, vp, i64, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]
        L.orc_p2q.restype = i64
        L.orc_normalize.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_c2n.argtypes = [vp, vp, vp, vp, vp, vp]
        L.orc_dirichlet.argtypes = [vp, i32, vp, vp, vp, vp]
        L.orc_stretch.argtypes = [vp, d, d, vp]
        L.orc_nh_tau.argtypes = [vp, d, d, vp]
        L.orc_nh_tau.restype = C.c_int
        L.orc_nh_psi.argtypes = [vp, d, d]
        L.orc_nh_psi.restype = d
        L.orc_nh_stretch.argtypes = [vp, d, d, vp, vp]
        L.orc_nh_stretch.restype = C.c_int
        L.orc_nh_cardano.argtypes = [d, d, d, vp]
        L.orc_nh_cardano.restype = d
        L.orc_stretch_all.argtypes = [vp, i32, vp, vp, vp, vp]
        L.orc_energy.argtypes = [vp, vp]
        L.orc_energy.restype = d
        L.orc_gradient.argtypes = [vp, vp, vp]
        L.orc_hvp.argtypes = [vp, vp, vp, vp]
        L.orc_diag.argtypes = [vp, vp, vp]
        L.orc_newton.argtypes = [vp, vp, vp, vp]
        L.orc_g2p.argtypes = [vp, d, vp, vp, i64, vp, vp, vp, vp, i32]
        L.orc_g2p.restype = i64
        L.orc_g2p_mat.argtypes = [vp, d, vp, vp, i64, vp, vp, vp, vp, vp, vp, i32]
        L.orc_g2p_mat.restype = i64
        L.orc_water_pi.argtypes = [d, d]
        L.orc_water_pi.restype = d
        L.orc_water_psi_J.argtypes = [d, d]
        L.orc_water_psi_J.restype = d
        L.orc_water_jbase.argtypes = [d, d]
        L.orc_water_jbase.restype = d
        L.orc_water_tau.argtypes = [vp, d, vp]
        L.orc_water_tau.restype = C.c_int
        L.orc_water_psi.argtypes = [vp, d]
        L.orc_water_psi.restype = d
        L.orc_water_stretch.argtypes = [vp, d, vp]
        L.orc_vm_plastic_P.argtypes = [vp, d, d, vp]
        L.orc_vm_plastic_P.restype = C.c_int
        L.orc_vm_return.argtypes = [vp, d, d, vp]
        L.orc_plastic_update.argtypes = [vp, vp, vp, vp]
        L.orc_plastic_update.restype = i64
        L.orc_explicit_force.argtypes = [vp, i32, vp, vp, vp, vp]
        L.orc_psd_project9.argtypes = [vp, vp]
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclasses.dataclass
class Grid:
    n: Sequence[int]
    dx: float
    origin: Sequence[float] = (0.0, 0.0, 0.0)

    def c(self) -> _Grid:
        g = _Grid()
        for a in range(3):
            g.n[a] = int(self.n[a])
            g.origin[a] = float(self.origin[a])
        g.dx = float(self.dx)
        return g

    @property
    def ncells(self) -> int:
        return int(self.n[0]) * int(self.n[1]) * int(self.n[2])

    @property
    def nnodes(self) -> int:
        return (int(self.n[0]) + 1) * (int(self.n[1]) + 1) * (int(self.n[2]) + 1)

    def node_ijk(self) -> np.ndarray:
        g = np.meshgrid(*[np.arange(int(self.n[a]) + 1) for a in range(3)], indexing="ij")
        return np.stack([x.ravel() for x in g], 1)

    def cell_ijk(self) -> np.ndarray:
        g = np.meshgrid(*[np.arange(int(self.n[a])) for a in range(3)], indexing="ij")
        return np.stack([x.ravel() for x in g], 1)


def _mats(materials) -> "C.Array":
    arr = (_Mat * MAXMAT)()
    for k, m in enumerate(materials):
        arr[k].E, arr[k].nu, arr[k].rho = float(m.E), float(m.nu), float(m.rho)
        arr[k].kind = int(getattr(m, "kind", 0))  # 0 StVK-Hencky, 1 split Neo-Hookean, 2 water (kappa = E)
        arr[k].yield_stress = float(getattr(m, "yield_stress", 0.0))  # von Mises sigma_y (kind 0; 0 = elastic)
    return arr


def lame(E: float, nu: float):
    """Standard 3D Lamé parameters (amb-2), written out independently of the GPU library."""
    return E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))


# ---------------------------------------------------------------------------------------------
# C1-C5: unload (Alg. 2) and stretch bases (Alg. 3 lines 4-7)
# ---------------------------------------------------------------------------------------------

def base_cells(grid: Grid, x: np.ndarray) -> np.ndarray:
    x = _f64(x)
    out = np.zeros((x.shape[0], 3), np.int32)
    lib().orc_base_cells(C.byref(grid.c()), x.shape[0], _p(x), _p(out))
    return out


def structural_cells(grid: Grid, base: np.ndarray) -> np.ndarray:
    """C1: the union of every particle's 2^3 stencil (cells b + o, o in {0,1}^3), as sorted
    x-major dense cell ids."""
    base = np.asarray(base, np.int64)
    n1, n2 = int(grid.n[1]), int(grid.n[2])
    ids = []
    for o in range(8):
        c = base + np.array([(o >> 2) & 1, (o >> 1) & 1, o & 1])
        ids.append((c[:, 0] * n1 + c[:, 1]) * n2 + c[:, 2])
    return np.unique(np.concatenate(ids))


def active_blocks(grid: Grid, base: np.ndarray) -> np.ndarray:
    """C1: sorted x-major ids (bx*NBy + by)*NBz + bz of the 4^3 cell blocks holding a stencil cell."""
    n1, n2 = int(grid.n[1]), int(grid.n[2])
    ids = structural_cells(grid, base)
    c = np.stack([ids // (n1 * n2), (ids // n2) % n1, ids % n2], 1)
    nb = [(int(grid.n[a]) + 3) // 4 for a in range(3)]
    b = c // 4
    return np.unique((b[:, 0] * nb[1] + b[:, 1]) * nb[2] + b[:, 2])


def q1_weights(f) -> np.ndarray:
    f = _f64(f)
    w = np.zeros(8)
    lib().orc_q1_weights(_p(f), _p(w))
    return w


def sym_eig3(A) -> tuple:
    A = _f64(A).reshape(9)
    w, Q = np.zeros(3), np.zeros(9)
    lib().orc_sym_eig3(_p(A), _p(w), _p(Q))
    return w, Q.reshape(3, 3)


def hencky_tau(F, mu: float, lam: float) -> np.ndarray:
    F = _f64(F).reshape(9)
    t = np.zeros(9)
    if lib().orc_hencky_tau(_p(F), mu, lam, _p(t)) != 0:
        raise ValueError("inverted F (det <= 0)")
    return t.reshape(3, 3)


def hencky_psi(F, mu: float, lam: float) -> float:
    F = _f64(F).reshape(9)
    return float(lib().orc_hencky_psi(_p(F), mu, lam))


def bulk_modulus(mu: float, lam: float) -> float:
    """kappa = 2/3 mu + lam in 3D."""
    return 2.0 * mu / 3.0 + lam


def nh_tau(F, mu: float, kappa: float) -> np.ndarray:
    """Split Neo-Hookean Kirchhoff stress (Eq. split-nh-tau)."""
    F = _f64(F).reshape(9)
    t = np.zeros(9)
    if lib().orc_nh_tau(_p(F), mu, kappa, _p(t)) != 0:
        raise ValueError("inverted F (det <= 0)")
    return t.reshape(3, 3)


def nh_psi(F, mu: float, kappa: float) -> float:
    """Split Neo-Hookean energy density (Eq. split-nh-energy)."""
    F = _f64(F).reshape(9)
    return float(lib().orc_nh_psi(_p(F), mu, kappa))


def nh_stretch(tau, mu: float, kappa: float):
    """Split Neo-Hookean stretch reconstruction (App. C Cardano); returns (S, branch)
    with branch 1 (Delta >= 0) or 3 (three real roots)."""
    tau = _f64(tau).reshape(9)
    S = np.zeros(9)
    br = C.c_int32(0)
    if lib().orc_nh_stretch(_p(tau), mu, kappa, _p(S), C.byref(br)) != 0:
        raise ValueError("stress outside the split Neo-Hookean inversion domain")
    return S.reshape(3, 3), br.value


def nh_cardano(p: float, q: float, dmin: float):
    br = C.c_int32(0)
    m = lib().orc_nh_cardano(float(p), float(q), float(dmin), C.byref(br))
    return m, br.value


def water_pi(J: float, kappa: float) -> float:
    """Water Kirchhoff pressure pi(J) = J psi'(J) = kappa J (J - 1) (§4.5)."""
    return float(lib().orc_water_pi(float(J), float(kappa)))


def water_psi_J(J: float, kappa: float) -> float:
    """Water energy density psi(J) = kappa/2 (J - 1)^2."""
    return float(lib().orc_water_psi_J(float(J), float(kappa)))


def water_jbase(pi: float, kappa: float) -> float:
    """J_base = (1 + sqrt(1 + 4 pi / kappa)) / 2, radicand clamped at 0."""
    return float(lib().orc_water_jbase(float(pi), float(kappa)))


def water_tau(F, kappa: float) -> np.ndarray:
    F = _f64(F).reshape(9)
    t = np.zeros(9)
    if lib().orc_water_tau(_p(F), kappa, _p(t)) != 0:
        raise ValueError("inverted F (det <= 0)")
    return t.reshape(3, 3)


def water_psi(F, kappa: float) -> float:
    F = _f64(F).reshape(9)
    return float(lib().orc_water_psi(_p(F), kappa))


def water_stretch(tau, kappa: float) -> np.ndarray:
    """Base stretch of a water slot: J_base(tr tau / 3)^{1/3} I."""
    tau = _f64(tau).reshape(9)
    S = np.zeros(9)
    lib().orc_water_stretch(_p(tau), kappa, _p(S))
    return S.reshape(3, 3)


def vm_plastic_P(F, mu: float, sigma_y: float):
    """Von Mises return map in Hencky space as F^E = F P: (P, projected)."""
    F = _f64(F).reshape(9)
    P = np.zeros(9)
    r = lib().orc_vm_plastic_P(_p(F), float(mu), float(sigma_y), _p(P))
    return P.reshape(3, 3), bool(r)


def vm_return(F, mu: float, sigma_y: float) -> np.ndarray:
    F = _f64(F).reshape(9)
    FE = np.zeros(9)
    lib().orc_vm_return(_p(F), float(mu), float(sigma_y), _p(FE))
    return FE.reshape(3, 3)


def stretch(tau, mu: float, lam: float) -> np.ndarray:
    tau = _f64(tau).reshape(9)
    S = np.zeros(9)
    lib().orc_stretch(_p(tau), mu, lam, _p(S))
    return S.reshape(3, 3)


@dataclasses.dataclass
class Unloaded:
    grid: Grid
    nmat: int
    m_c: np.ndarray
    mv_c: np.ndarray
    mG_c: np.ndarray
    V_ck: np.ndarray
    Vtau_ck: np.ndarray
    v_c: np.ndarray
    G_c: np.ndarray
    tau_ck: np.ndarray
    m_i: np.ndarray
    v_i: np.ndarray


def unload(grid: Grid, materials, x, v, F, G, vol, mat, clip: bool = False) -> Unloaded:
    """Alg. 2: P2C with stress content, normalisation, C2N gather."""
    x, v, F, G, vol = _f64(x), _f64(v), _f64(F), _f64(G), _f64(vol)
    mat = np.ascontiguousarray(mat, dtype=np.int32)
    nc, nn, nm = grid.ncells, grid.nnodes, len(materials)
    m_c, mv_c, mG_c = np.zeros(nc), np.zeros((nc, 3)), np.zeros((nc, 9))
    V_ck, Vtau_ck = np.zeros((nm, nc)), np.zeros((nm, nc, 9))
    g = grid.c()
    r = lib().orc_p2q(C.byref(g), nm, _mats(materials), x.shape[0], _p(x), _p(v), _p(F), _p(G), _p(vol),
                      _p(mat), int(clip), _p(m_c), _p(mv_c), _p(mG_c), _p(V_ck), _p(Vtau_ck))
    if r != 0:
        raise ValueError(f"oracle p2q: particle {-r - 1} out of domain or inverted")
    v_c, G_c, tau_ck = np.zeros((nc, 3)), np.zeros((nc, 9)), np.zeros((nm, nc, 9))
    lib().orc_normalize(C.byref(g), nm, _p(m_c), _p(mv_c), _p(mG_c), _p(V_ck), _p(Vtau_ck), _p(v_c),
                        _p(G_c), _p(tau_ck))
    m_i, v_i = np.zeros(nn), np.zeros((nn, 3))
    lib().orc_c2n(C.byref(g), _p(m_c), _p(v_c), _p(G_c), _p(m_i), _p(v_i))
    return Unloaded(grid, nm, m_c, mv_c, mG_c, V_ck, Vtau_ck, v_c, G_c, tau_ck, m_i, v_i)


def stretch_bases(grid: Grid, materials, V_ck, tau_ck) -> np.ndarray:
    """Alg. 3 lines 4-7: S_{c,k} from tau_{c,k} where V_{c,k} != 0 (identity elsewhere)."""
    nm = len(materials)
    V_ck, tau_ck = _f64(V_ck), _f64(tau_ck)
    S = np.zeros((nm, grid.ncells, 9))
    lib().orc_stretch_all(C.byref(grid.c()), nm, _mats(materials), _p(V_ck), _p(tau_ck), _p(S))
    return S


def dirichlet(grid: Grid, boxes, m_i) -> tuple:
    nb = len(boxes)
    arr = (_Box * max(nb, 1))()
    for b, bx in enumerate(boxes):
        for a in range(3):
            arr[b].lo[a], arr[b].hi[a], arr[b].vel[a] = bx.lo[a], bx.hi[a], bx.velocity[a]
    freed = np.zeros(grid.nnodes, np.uint8)
    vfix = np.zeros((grid.nnodes, 3))
    m_i = _f64(m_i)
    lib().orc_dirichlet(C.byref(grid.c()), nb, arr, _p(m_i), _p(freed), _p(vfix))
    return freed, vfix


# ---------------------------------------------------------------------------------------------
# C6-C7: the incremental potential and its Newton-PCG minimisation
# ---------------------------------------------------------------------------------------------

class Problem:
    """Integrate-time problem (Alg. 3): everything the solve reads, nothing from particles."""

    def __init__(self, grid: Grid, materials, dt: float, m_i, vhat, freed, m_c, V_ck, S_ck, psd: bool = False):
        self.grid, self.materials, self.dt = grid, list(materials), float(dt)
        self.psd = bool(psd)  # Hessian blocks K_c PSD-projected: hvp, diag and the Newton solve
        self.m_i, self.vhat = _f64(m_i), _f64(vhat).reshape(-1, 3)
        self.freed = np.ascontiguousarray(freed, dtype=np.uint8)
        self.m_c, self.V_ck, self.S_ck = _f64(m_c), _f64(V_ck), _f64(S_ck)
        P = _Problem()
        P.g = grid.c()
        P.nmat = len(materials)
        P.mats = _mats(materials)
        P.dt = self.dt
        P.m_i, P.vhat, P.freed = _p(self.m_i).value, _p(self.vhat).value, _p(self.freed).value
        P.m_c, P.V_ck, P.S_ck = _p(self.m_c).value, _p(self.V_ck).value, _p(self.S_ck).value
        P.psd = int(self.psd)
        self._c = P

    def plastic_update(self, v):
        """Bases after the von Mises return map at iterate v: (S_ck, number of projected slots)."""
        v = _f64(v).reshape(-1, 3)
        S = np.zeros_like(self.S_ck)
        n = lib().orc_plastic_update(C.byref(self._c), _p(v), _p(self.S_ck), _p(S))
        return S, int(n)

    def with_bases(self, S_ck) -> "Problem":
        """The same problem with other bases (e.g. the plastic iterate's, held fixed)."""
        return Problem(self.grid, self.materials, self.dt, self.m_i, self.vhat, self.freed, self.m_c, self.V_ck, S_ck,
                       self.psd)

    def with_psd(self, psd: bool) -> "Problem":
        """The same problem with the exact (False) or per-cell PSD-projected (True) Hessian."""
        return Problem(self.grid, self.materials, self.dt, self.m_i, self.vhat, self.freed, self.m_c, self.V_ck,
                       self.S_ck, psd)

    def energy(self, v) -> float:
        v = _f64(v).reshape(-1, 3)
        return float(lib().orc_energy(C.byref(self._c), _p(v)))

    def gradient(self, v) -> np.ndarray:
        v = _f64(v).reshape(-1, 3)
        g = np.zeros_like(v)
        lib().orc_gradient(C.byref(self._c), _p(v), _p(g))
        return g

    def hvp(self, v, u) -> np.ndarray:
        v, u = _f64(v).reshape(-1, 3), _f64(u).reshape(-1, 3)
        out = np.zeros_like(v)
        lib().orc_hvp(C.byref(self._c), _p(v), _p(u), _p(out))
        return out

    def diag(self, v) -> np.ndarray:
        v = _f64(v).reshape(-1, 3)
        out = np.zeros_like(v)
        lib().orc_diag(C.byref(self._c), _p(v), _p(out))
        return out

    def newton(self, v0, solver, fixed_newton: int = 0, fixed_cg: Optional[Sequence[int]] = None,
               fixed_ls: Optional[Sequence[int]] = None):
        if bool(getattr(solver, "psd", False)) != self.psd:  # the solver's Hessian mode
            return self.with_psd(bool(getattr(solver, "psd", False))).newton(v0, solver, fixed_newton, fixed_cg, fixed_ls)
        v = _f64(v0).reshape(-1, 3).copy()
        cfg = _SolverCfg()
        cfg.newton_max, cfg.cg_max, cfg.ls_max = solver.newton_max, solver.cg_max, solver.ls_max
        cfg.eps_newton, cfg.eps_cg, cfg.armijo = solver.eps_newton, solver.eps_cg, solver.armijo
        cfg.fixed_newton = int(fixed_newton)
        fc = None
        if fixed_cg is not None:
            fc = np.ascontiguousarray(fixed_cg, dtype=np.int32)
            cfg.fixed_cg = _p(fc).value
        fl = None
        if fixed_ls is not None:
            fl = np.ascontiguousarray(fixed_ls, dtype=np.int32)
            cfg.fixed_ls = _p(fl).value
        cfg.ls_slack = float(getattr(solver, "ls_slack", 1e-13))
        st = _Stats()
        lib().orc_newton(C.byref(self._c), C.byref(cfg), _p(v), C.byref(st))
        n = st.newton_iters
        stats = dict(newton_iters=n, cg_total=st.cg_total, ls_halvings=st.ls_halvings,
                     converged=st.converged, neg_curv=st.neg_curv, grad_norm0=st.grad_norm0,
                     grad_norm=st.grad_norm, energy=st.energy,
                     cg_iters=[st.cg_iters[k] for k in range(min(n, 64))],
                     ls_iters=[st.ls_iters[k] for k in range(min(n, 64))])
        return v, stats


def psd_project9(M) -> np.ndarray:
    """Per-cell PSD projection of a symmetric 9x9 block: Q max(Lambda, 0) Q^T (oracle's cyclic Jacobi)."""
    M = _f64(M).reshape(81)
    out = np.zeros(81)
    lib().orc_psd_project9(_p(M), _p(out))
    return out.reshape(9, 9)


def explicit_force(grid: Grid, nmat: int, m_c, V_ck, tau_ck) -> np.ndarray:
    f = np.zeros((grid.nnodes, 3))
    lib().orc_explicit_force(C.byref(grid.c()), nmat, _p(_f64(m_c)), _p(_f64(V_ck)), _p(_f64(tau_ck)), _p(f))
    return f


def g2p(grid: Grid, dt: float, m_c, v_i, x, v, F, G, clip: bool = False, mat=None, materials=None):
    """Alg. 4. Returns updated copies (x, v, F, G).  With (mat, materials), water
    particles (kind 2) update J_p by the trace form of P:316 and keep F_p = J_p^{1/3} I."""
    x, v, F, G = _f64(x).copy(), _f64(v).copy(), _f64(F).copy(), _f64(G).copy()
    if mat is not None and any(getattr(m, "kind", 0) == 2 or getattr(m, "yield_stress", 0.0) > 0 for m in materials):
        mat = np.ascontiguousarray(mat, dtype=np.int32)
        r = lib().orc_g2p_mat(C.byref(grid.c()), float(dt), _p(_f64(m_c)), _p(_f64(v_i).reshape(-1, 3)),
                              x.shape[0], _p(x), _p(v), _p(F), _p(G), _p(mat), _mats(materials), int(clip))
    else:
        r = lib().orc_g2p(C.byref(grid.c()), float(dt), _p(_f64(m_c)), _p(_f64(v_i).reshape(-1, 3)), x.shape[0],
                          _p(x), _p(v), _p(F), _p(G), int(clip))
    if r != 0:
        raise ValueError(f"oracle g2p: particle {-r - 1} out of domain")
    return x, v, F, G


# ---------------------------------------------------------------------------------------------
# Alg. 1: one full step, composed from the pieces above
# ---------------------------------------------------------------------------------------------

@dataclasses.dataclass
class StepResult:
    unloaded: Unloaded
    S_ck: np.ndarray
    problem: Problem
    v0: np.ndarray
    v_new: np.ndarray
    stats: dict
    particles: tuple  # (x, v, F, G) after Load


def prepare(scene, grid: Optional[Grid] = None, clip: bool = False):
    """Unload + stretch bases + Dirichlet sets + Newton start v0 (amb-4, amb-9)."""
    grid = grid or Grid(scene.n, scene.dx, scene.origin)
    un = unload(grid, scene.materials, scene.x, scene.v, scene.F, scene.G, scene.vol, scene.mat, clip)
    S = stretch_bases(grid, scene.materials, un.V_ck, un.tau_ck)
    gvec = np.asarray(scene.gravity, dtype=np.float64)
    vhat = un.v_i + scene.dt * gvec[None, :] * (un.m_i[:, None] > 0)
    freed, vfix = dirichlet(grid, scene.dirichlet, un.m_i)
    fixed = (un.m_i > 0) & (freed == 0)
    v0 = np.where(fixed[:, None], vfix, vhat)
    v0[un.m_i == 0] = 0.0
    prob = Problem(grid, scene.materials, scene.dt, un.m_i, vhat, freed, un.m_c, un.V_ck, S)
    return un, S, prob, v0


def step(scene, fixed_newton: int = 0, fixed_cg=None, solver=None, fixed_ls=None) -> StepResult:
    un, S, prob, v0 = prepare(scene)
    vnew, stats = prob.newton(v0, solver or scene.solver, fixed_newton, fixed_cg, fixed_ls)
    parts = g2p(prob.grid, scene.dt, un.m_c, vnew, scene.x, scene.v, scene.F, scene.G, mat=scene.mat,
                materials=scene.materials)
    return StepResult(un, S, prob, v0, vnew, stats, parts)
