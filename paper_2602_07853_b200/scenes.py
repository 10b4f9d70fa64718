"""Seeded synthetic scenes (BASELINE.json configs 1-5) — INPUT GENERATORS ONLY.

This module is shared by the CUDA path's tests/bench and by the CPU oracle's
tests.  It holds none of the method's arithmetic (no weights, no transfers, no
constitutive law): it only lays out particles, initial velocities, material
parameters, Dirichlet boxes and solver settings as plain arrays.  The recipe
for every config is stated in DESIGN.md §3 (input recipe) and follows
SURVEY.md §8(d), with the readings amb-11..amb-17 of SURVEY.md §8(c).

Seeds: 0 jitter, 1 velocity noise, 2 smooth-field draws,
3 pre-strain, 4 HVP direction, 5 gradient probe.

Geometry convention: domain [0,1]^3, origin 0, N^3 cells, dx = 1/N (a power
of two in every config, so x/dx - 1/2 is exact in fp32 and fp64).  A cell is
"filled" when its centre lies inside the shape (voxelisation); every filled
cell receives PPC = k^3 stratified particles (one uniform point per sub-cell,
amb-11).  Rest volume V_p = dx^3/PPC; mass is rho_k * V_p and is
formed by each side from the material table.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

GRAVITY = (0.0, -9.81, 0.0)  # amb-4: y up


@dataclasses.dataclass
class Material:
    E: float
    nu: float
    rho: float
    kind: int = 0  # 0 StVK-Hencky, 1 split Neo-Hookean, 2 water (kappa = E)
    yield_stress: float = 0.0  # von Mises sigma_y for kind 0 (fixed-point plasticity); 0 = elastic


@dataclasses.dataclass
class DirichletBox:
    lo: Tuple[float, float, float]
    hi: Tuple[float, float, float]
    velocity: Tuple[float, float, float]


@dataclasses.dataclass
class SolverCfg:
    eps_cg: float = 1e-5
    eps_newton: float = 1e-5
    newton_max: int = 10
    cg_max: int = 10000
    ls_max: int = 30
    armijo: float = 1e-4
    ls_slack: float = 1e-13  # Armijo rounding slack relative to |Phi| (amb-6); fp32 runs use 1e-6
    psd: bool = False  # per-cell PSD projection of the Hessian; cfg5 (indefinite under the plate)


@dataclasses.dataclass
class Scene:
    name: str
    precision: int  # 32 or 64
    n: Tuple[int, int, int]
    dx: float
    dt: float
    materials: List[Material]
    x: np.ndarray  # (np,3)
    v: np.ndarray  # (np,3)
    F: np.ndarray  # (np,9) row-major
    G: np.ndarray  # (np,9) row-major
    vol: np.ndarray  # (np,)
    mat: np.ndarray  # (np,) int32
    dirichlet: List[DirichletBox]
    solver: SolverCfg
    steps: int = 1
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    gravity: Tuple[float, float, float] = GRAVITY

    @property
    def n_particles(self) -> int:
        return int(self.x.shape[0])

    @property
    def dtype(self):
        return np.float32 if self.precision == 32 else np.float64


# ----------------------------------------------------------------------------
# voxelised shapes: return (m,3) int arrays of filled cells (x-major order)
# ----------------------------------------------------------------------------

def _centres(n: int, lo: int, hi: int) -> np.ndarray:
    return (np.arange(lo, hi) + 0.5) / n


def cells_box(lo: Sequence[int], hi: Sequence[int]) -> np.ndarray:
    gx, gy, gz = np.meshgrid(np.arange(lo[0], hi[0]), np.arange(lo[1], hi[1]),
                             np.arange(lo[2], hi[2]), indexing="ij")
    return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1).astype(np.int64)


def cells_sphere(n: int, centre, radius) -> np.ndarray:
    lo = [max(0, int(math.floor((centre[a] - radius) * n)) - 1) for a in range(3)]
    hi = [min(n, int(math.ceil((centre[a] + radius) * n)) + 1) for a in range(3)]
    c = cells_box(lo, hi)
    xc = (c + 0.5) / n
    d2 = ((xc - np.asarray(centre)) ** 2).sum(1)
    return c[d2 < radius * radius]


def cells_slab(n: int, xlo, xhi, ylo, yhi, zlo, zhi) -> np.ndarray:
    def rng_idx(a, b):
        i = np.arange(n)
        xc = (i + 0.5) / n
        return i[(xc >= a) & (xc < b)]
    ix, iy, iz = rng_idx(xlo, xhi), rng_idx(ylo, yhi), rng_idx(zlo, zhi)
    gx, gy, gz = np.meshgrid(ix, iy, iz, indexing="ij")
    return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1).astype(np.int64)


def cells_wheel(n: int, centre, r_out, r_in, width) -> np.ndarray:
    """Annulus around an axis parallel to z (cfg5)."""
    lo = [max(0, int(math.floor((centre[0] - r_out) * n)) - 1),
          max(0, int(math.floor((centre[1] - r_out) * n)) - 1),
          max(0, int(math.floor((centre[2] - width / 2) * n)) - 1)]
    hi = [min(n, int(math.ceil((centre[0] + r_out) * n)) + 1),
          min(n, int(math.ceil((centre[1] + r_out) * n)) + 1),
          min(n, int(math.ceil((centre[2] + width / 2) * n)) + 1)]
    out = []
    # slice along x to bound memory
    for ix in range(lo[0], hi[0]):
        c = cells_box([ix, lo[1], lo[2]], [ix + 1, hi[1], hi[2]])
        xc = (c + 0.5) / n
        rr = (xc[:, 0] - centre[0]) ** 2 + (xc[:, 1] - centre[1]) ** 2
        keep = (rr <= r_out * r_out) & (rr >= r_in * r_in) & (np.abs(xc[:, 2] - centre[2]) <= width / 2)
        out.append(c[keep])
    return np.concatenate(out, 0)


def unique_cells(*arrs: np.ndarray) -> np.ndarray:
    c = np.concatenate(arrs, 0)
    c = np.unique(c, axis=0)  # sorted x-major
    return c


# ----------------------------------------------------------------------------
# stratified jitter (amb-11): PPC = k^3, one uniform point per sub-cell
# ----------------------------------------------------------------------------

def stratified(cells: np.ndarray, n: int, k: int, seed: int = 0, dtype=np.float64,
               chunk: int = 1 << 18) -> np.ndarray:
    rng = np.random.default_rng(seed)
    dx = 1.0 / n
    ppc = k ** 3
    s = cells_box([0, 0, 0], [k, k, k]).astype(np.float64)  # (ppc,3) x-major sub-cells
    out = np.empty((cells.shape[0] * ppc, 3), dtype=dtype)
    for c0 in range(0, cells.shape[0], chunk):
        c = cells[c0:c0 + chunk].astype(np.float64)
        u = rng.random((c.shape[0], ppc, 3))
        pos = dx * (c[:, None, :] + (s[None, :, :] + u) / k)
        out[c0 * ppc:(c0 + c.shape[0]) * ppc] = pos.reshape(-1, 3)
    return out


def smooth_field(seed: int = 2):
    """Sum of 8 sinusoids (amb-12/cfg2): v(x) = sum_k a_k sin(2 pi n_k.x + phi_k)."""
    rng = np.random.default_rng(seed)
    nk = rng.integers(1, 4, size=(8, 3)).astype(np.float64)
    ak = rng.normal(0.0, 0.1, size=(8, 3))
    ph = rng.uniform(0.0, 2 * math.pi, size=8)
    return nk, ak, ph


def eval_smooth_field(x: np.ndarray, field, chunk: int = 1 << 20):
    """Velocity and its analytic gradient G_ab = dv_a/dx_b at x (float64)."""
    nk, ak, ph = field
    v = np.zeros((x.shape[0], 3))
    G = np.zeros((x.shape[0], 9))
    for i0 in range(0, x.shape[0], chunk):
        xx = x[i0:i0 + chunk].astype(np.float64)
        arg = 2 * math.pi * xx @ nk.T + ph[None, :]  # (m,8)
        s, c = np.sin(arg), np.cos(arg)
        v[i0:i0 + chunk] = s @ ak
        # G_ab = sum_k a_ka * cos * 2 pi n_kb
        G[i0:i0 + chunk] = np.einsum("mk,ka,kb->mab", c, ak, 2 * math.pi * nk).reshape(-1, 9)
    return v, G


def _identity(np_: int, dtype) -> np.ndarray:
    F = np.zeros((np_, 9), dtype=dtype)
    F[:, 0] = F[:, 4] = F[:, 8] = 1
    return F


def _prestrain(np_: int, seed: int = 3) -> np.ndarray:
    """amb-17 cfg1b: F_p = R_p (I + 0.05 Y_p), Y symmetric N(0,1), R axis-uniform, angle U[0,pi/6]."""
    rng = np.random.default_rng(seed)
    up = rng.normal(size=(np_, 6))
    Y = np.zeros((np_, 3, 3))
    Y[:, 0, 0], Y[:, 1, 1], Y[:, 2, 2] = up[:, 0], up[:, 1], up[:, 2]
    Y[:, 0, 1] = Y[:, 1, 0] = up[:, 3]
    Y[:, 1, 2] = Y[:, 2, 1] = up[:, 4]
    Y[:, 0, 2] = Y[:, 2, 0] = up[:, 5]
    axis = rng.normal(size=(np_, 3))
    axis /= np.linalg.norm(axis, axis=1, keepdims=True)
    ang = rng.uniform(0.0, math.pi / 6, size=np_)
    Kx = np.zeros((np_, 3, 3))
    Kx[:, 0, 1], Kx[:, 0, 2] = -axis[:, 2], axis[:, 1]
    Kx[:, 1, 0], Kx[:, 1, 2] = axis[:, 2], -axis[:, 0]
    Kx[:, 2, 0], Kx[:, 2, 1] = -axis[:, 1], axis[:, 0]
    s, c = np.sin(ang)[:, None, None], np.cos(ang)[:, None, None]
    R = np.eye(3)[None] + s * Kx + (1 - c) * (Kx @ Kx)  # Rodrigues
    F = R @ (np.eye(3)[None] + 0.05 * Y)
    return F.reshape(-1, 9)


def _assemble(name, precision, n, dt, materials, x, v, F, G, mat, ppc, dirichlet, solver, steps):
    dt_ = np.float32 if precision == 32 else np.float64
    dx = 1.0 / n
    vol = np.full(x.shape[0], dx ** 3 / ppc, dtype=dt_)
    if precision == 32:  # Phi is resolved to ~1e-7 relative in fp32 (amb-6 slack)
        solver = dataclasses.replace(solver, ls_slack=max(solver.ls_slack, 1e-6))
    return Scene(name=name, precision=precision, n=(n, n, n), dx=dx, dt=dt, materials=materials,
                 x=np.ascontiguousarray(x, dtype=dt_), v=np.ascontiguousarray(v, dtype=dt_),
                 F=np.ascontiguousarray(F, dtype=dt_), G=np.ascontiguousarray(G, dtype=dt_),
                 vol=vol, mat=np.ascontiguousarray(mat, dtype=np.int32), dirichlet=dirichlet,
                 solver=solver, steps=steps)


# ----------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------

def cfg1(prestrain: bool = False, precision: int = 64) -> Scene:
    """Tiny elastic cube: 16^3, cells [4,12)^3, 8 PPC (4096 particles), E=1e4 nu=0.3 rho=1000."""
    n = 16
    cells = cells_box([4, 4, 4], [12, 12, 12])
    x = stratified(cells, n, 2, seed=0)
    v = np.random.default_rng(1).normal(0.0, 0.1, size=(x.shape[0], 3))
    F = _prestrain(x.shape[0]) if prestrain else _identity(x.shape[0], np.float64)
    G = np.zeros((x.shape[0], 9))
    tol = (1e-8, 1e-9) if precision == 64 else (1e-5, 1e-5)
    return _assemble("cfg1b" if prestrain else "cfg1", precision, n, 1e-3, [Material(1e4, 0.3, 1000.0)],
                     x, v, F, G, np.zeros(x.shape[0], np.int32), 8, [],
                     SolverCfg(eps_cg=tol[0], eps_newton=tol[1]), 1)


def cfg2(precision: int = 32) -> Scene:
    """Dense block: 64^3, cells [8,56)^3, 8 PPC, E=1e5 nu=0.4, smooth sinusoid velocity, dt=2e-3."""
    n = 64
    cells = cells_box([8, 8, 8], [56, 56, 56])
    x = stratified(cells, n, 2, seed=0, dtype=np.float32 if precision == 32 else np.float64)
    v, G = eval_smooth_field(x, smooth_field(2))
    tol = (1e-8, 1e-9) if precision == 64 else (1e-5, 1e-5)
    return _assemble("cfg2", precision, n, 2e-3, [Material(1e5, 0.4, 1000.0)], x, v,
                     _identity(x.shape[0], np.float64), G, np.zeros(x.shape[0], np.int32), 8, [],
                     SolverCfg(eps_cg=tol[0], eps_newton=tol[1]), 10)


def cfg3(ppc_k: int = 2, precision: int = 32) -> Scene:
    """PPC sweep: 128^3, cells [8,120)^3, PPC = k^3 in {1,8,27,64}, E=1e6 nu=0.3, cfg2's field."""
    n = 128
    cells = cells_box([8, 8, 8], [120, 120, 120])
    x = stratified(cells, n, ppc_k, seed=0, dtype=np.float32 if precision == 32 else np.float64)
    v, G = eval_smooth_field(x, smooth_field(2))
    return _assemble(f"cfg3_ppc{ppc_k ** 3}", precision, n, 1e-3, [Material(1e6, 0.3, 1000.0)], x, v,
                     _identity(x.shape[0], np.float64), G, np.zeros(x.shape[0], np.int32), ppc_k ** 3, [],
                     SolverCfg(), 3)


def cfg4(precision: int = 32, n: int = 256) -> Scene:
    """Sparse collision: 256^3, two spheres r=0.2 approaching at +-1 m/s + ground slab, 8 PPC.

    Spheres: E=5e4 nu=0.35 (material 0); slab y in [3dx,16dx), x,z in [3dx,1-3dx): E=1e7 nu=0.35
    (material 1); rho=1000; sticky floor: nodes with y <= 3dx fixed at v=0.
    """
    dx = 1.0 / n
    dt_ = np.float32 if precision == 32 else np.float64
    s0 = cells_sphere(n, (0.25, 0.35, 0.5), 0.2)
    s1 = cells_sphere(n, (0.75, 0.35, 0.5), 0.2)
    slab = cells_slab(n, 3 * dx, 1 - 3 * dx, 3 * dx, 16 * dx, 3 * dx, 1 - 3 * dx)
    xs0 = stratified(s0, n, 2, seed=0, dtype=dt_)
    xs1 = stratified(s1, n, 2, seed=10, dtype=dt_)
    xsl = stratified(slab, n, 2, seed=20, dtype=dt_)
    x = np.concatenate([xs0, xs1, xsl], 0)
    v = np.zeros((x.shape[0], 3), dtype=dt_)
    v[:xs0.shape[0], 0] = 1.0
    v[xs0.shape[0]:xs0.shape[0] + xs1.shape[0], 0] = -1.0
    mat = np.zeros(x.shape[0], np.int32)
    mat[xs0.shape[0] + xs1.shape[0]:] = 1
    inf = float("inf")
    floor = DirichletBox((-inf, -inf, -inf), (inf, 3 * dx, inf), (0.0, 0.0, 0.0))
    return _assemble("cfg4", precision, n, 1e-3,
                     [Material(5e4, 0.35, 1000.0), Material(1e7, 0.35, 1000.0)],
                     x, v, _identity(x.shape[0], dt_), np.zeros((x.shape[0], 9), dt_), mat, 8, [floor],
                     SolverCfg(), 3)


def cfg5(variant: str = "B", precision: int = 32, n: int = 512) -> Scene:
    """Large stiff press: 512^3 annular wheel (R=0.3, r=0.1, width 0.15) under a plate moving at 0.5 m/s.

    E=7e10 nu=0.33 rho=2700.  Variant B (amb-14) adds a ground slab y in [3dx,29dx) of wheel material.
    """
    dx = 1.0 / n
    dt_ = np.float32 if precision == 32 else np.float64
    cy = (29 * dx if variant == "B" else 3 * dx) + 0.3
    parts = [cells_wheel(n, (0.5, cy, 0.5), 0.3, 0.1, 0.15)]
    if variant == "B":
        parts.append(cells_slab(n, 3 * dx, 1 - 3 * dx, 3 * dx, 29 * dx, 3 * dx, 1 - 3 * dx))
    cells = unique_cells(*parts)
    x = stratified(cells, n, 2, seed=0, dtype=dt_)
    inf = float("inf")
    floor = DirichletBox((-inf, -inf, -inf), (inf, 3 * dx, inf), (0.0, 0.0, 0.0))
    plate = DirichletBox((-inf, cy + 0.3, -inf), (inf, inf, inf), (0.0, -0.5, 0.0))
    # solver (DESIGN.md §2 amb-6c): the exact Hessian is indefinite under the plate (compressed cells: PCG
    # stops at negative curvature, the line search stalls), so per-cell PSD projection; Jacobi-PCG
    # at r = 1e7 reaches ||g|| <= 1e-4 ||g0|| within the 10^4 CG cap as an inexact Newton (eta = 1e-2),
    # not 1e-5 (measured: profiles/r02_cfg5_convergence.jsonl)
    return _assemble(f"cfg5{variant}", precision, n, 1e-3, [Material(7e10, 0.33, 2700.0)], x,
                     np.zeros((x.shape[0], 3), dt_), _identity(x.shape[0], dt_),
                     np.zeros((x.shape[0], 9), dt_), np.zeros(x.shape[0], np.int32), 8, [floor, plate],
                     SolverCfg(eps_cg=1e-2, eps_newton=1e-4, psd=True), 3)


def jelly(precision: int = 32, n: int = 256) -> Scene:
    """Explicit-path workload in the shape of Table 1's falling jelly: Delta x = 1/256,
    dt = 6e-5, StVK-Hencky E=5e3 nu=0.4 rho=1000; a 52^3-cell cube at 8 PPC (1,124,864 particles vs the
    paper's 1.14M) released at 1 m/s downward over a sticky floor (the jelly mesh is not available)."""
    dt_ = np.float32 if precision == 32 else np.float64
    lo = np.array([102, 40, 102])
    cells = cells_box(lo, lo + 52)
    x = stratified(cells, n, 2, seed=0, dtype=dt_)
    v = np.zeros((x.shape[0], 3), dtype=dt_)
    v[:, 1] = -1.0
    dx = 1.0 / n
    inf = float("inf")
    floor = DirichletBox((-inf, -inf, -inf), (inf, 3 * dx, inf), (0.0, 0.0, 0.0))
    return _assemble("jelly", precision, n, 6e-5, [Material(5e3, 0.4, 1000.0)], x, v,
                     _identity(x.shape[0], dt_), np.zeros((x.shape[0], 9), dt_), np.zeros(x.shape[0], np.int32),
                     8, [floor], SolverCfg(), 100)


def by_name(name: str, precision: Optional[int] = None) -> Scene:
    if name == "cfg1":
        return cfg1(False, precision or 64)
    if name == "cfg1b":
        return cfg1(True, precision or 64)
    if name == "cfg2":
        return cfg2(precision or 32)
    if name.startswith("cfg3"):
        k = {"cfg3": 2, "cfg3_ppc1": 1, "cfg3_ppc8": 2, "cfg3_ppc27": 3, "cfg3_ppc64": 4}[name]
        return cfg3(k, precision or 32)
    if name == "cfg4":
        return cfg4(precision or 32)
    if name in ("cfg5", "cfg5B"):
        return cfg5("B", precision or 32)
    if name == "cfg5A":
        return cfg5("A", precision or 32)
    if name == "jelly":
        return jelly(precision or 32)
    if name == "cfg4_nh":  # SURVEY f1 measured on cfg4's geometry: both materials split Neo-Hookean
        sc = cfg4(precision or 32)
        return dataclasses.replace(sc, name=name, materials=[dataclasses.replace(m, kind=1) for m in sc.materials])
    if name == "cfg4_vm":  # SURVEY f2 on cfg4's geometry: pre-strained spheres with von Mises sigma_y = 500 Pa
        sc = cfg4(precision or 32)
        sph = sc.mat == 0
        F = sc.F.copy()
        F[sph] = _prestrain(int(sph.sum()), 5).astype(F.dtype)
        m0 = dataclasses.replace(sc.materials[0], yield_stress=500.0)
        return dataclasses.replace(sc, name=name, F=F, materials=[m0, sc.materials[1]])
    if name == "cfg4_water":  # SURVEY f4 on cfg4's geometry: the left sphere is J-based water (kappa = E)
        sc = cfg4(precision or 32)
        m0 = dataclasses.replace(sc.materials[0], E=2e5, kind=2)
        return dataclasses.replace(sc, name=name, materials=[m0, sc.materials[1]])
    raise KeyError(name)


def random_direction(n: int, seed: int = 4, dtype=np.float64) -> np.ndarray:
    """HVP probe u ~ N(0,1) per DOF (seed 4)."""
    return np.random.default_rng(seed).normal(size=(n, 3)).astype(dtype)


def gradient_probe(n: int, seed: int = 5, scale: float = 0.01, dtype=np.float64) -> np.ndarray:
    """Gradient probe perturbation 0.01 N(0,1) per DOF (seed 5)."""
    return (scale * np.random.default_rng(seed).normal(size=(n, 3))).astype(dtype)


def subset(scene: Scene, keep: np.ndarray, name: Optional[str] = None) -> Scene:
    """Scene restricted to particles `keep` (bool mask or index array) — used for windows."""
    return dataclasses.replace(scene, name=name or scene.name, x=scene.x[keep], v=scene.v[keep],
                               F=scene.F[keep], G=scene.G[keep], vol=scene.vol[keep], mat=scene.mat[keep])


def key_noise(keys: np.ndarray, seed: int, dims: int = 3) -> np.ndarray:
    """Standard-normal numbers indexed by an integer key (e.g. a global node id), so a full-size
    run and an oracle window draw identical probe values for the same node (splitmix64 + Box-Muller)."""
    with np.errstate(over="ignore"):
        k = np.asarray(keys, dtype=np.uint64).reshape(-1, 1) * np.uint64(2 * dims) + np.arange(
            2 * dims, dtype=np.uint64)[None, :] + np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
        z = k + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    u1, u2 = u[:, :dims], u[:, dims:]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
