"""Thin Python binding of libmpmlite.so (include/mpmlite.h) — argument marshalling only.

Every numerical step runs in the CUDA kernels behind the C ABI.  There is no CPU fallback:
importing this module raises if the in-tree library is missing, and every call raises
``MplError`` on a non-zero status.  Buffers may be numpy arrays (host) or torch tensors
(host or CUDA); the library copies with cudaMemcpyDefault.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPL_LIB=dbg loads the bounds-checked debug build (MPL_DEBUG=1 python -m paper_2602_07853_b200.build)
LIB_PATH = os.path.join(_HERE, "libmpmlite_dbg.so" if os.environ.get("MPL_LIB") == "dbg" else "libmpmlite.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2602_07853_b200.build` "
                      "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

STATUS = {0: "MPL_OK", 1: "MPL_ERR_INVALID_ARG", 2: "MPL_ERR_STATE", 3: "MPL_ERR_OUT_OF_DOMAIN",
          4: "MPL_ERR_INVERTED", 5: "MPL_ERR_INVERSION_DOMAIN", 6: "MPL_ERR_NONFINITE", 7: "MPL_ERR_OOM",
          8: "MPL_ERR_CUDA", 9: "MPL_ERR_NCCL", 10: "MPL_ERR_UNSUPPORTED"}


class MplError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Grid(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("dx", C.c_double), ("origin", C.c_double * 3)]


class Material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double),
                ("yield_stress", C.c_double)]


class Config(C.Structure):
    _fields_ = [("precision", C.c_int32), ("device", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("loopback", C.c_void_p)]


class DirichletBox(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("velocity", C.c_double * 3)]


class SolverCfg(C.Structure):
    _fields_ = [("newton_max", C.c_int32), ("cg_max", C.c_int32), ("newton_rtol", C.c_double),
                ("cg_rtol", C.c_double), ("armijo_c", C.c_double), ("ls_max", C.c_int32),
                ("ls_slack", C.c_double), ("fixed_newton_iters", C.c_int32), ("fixed_cg_iters", C.c_void_p),
                ("fixed_ls_halvings", C.c_void_p), ("psd_project", C.c_int32)]


MAX_NEWTON_LOG = 64


class SolveStats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("cg_iters_total", C.c_int32), ("ls_halvings", C.c_int32),
                ("converged", C.c_int32), ("neg_curvature", C.c_int32), ("n_inverted_trials", C.c_int32),
                ("grad_norm0", C.c_double), ("grad_norm", C.c_double), ("energy", C.c_double),
                ("cg_iters", C.c_int32 * MAX_NEWTON_LOG), ("ls_iters", C.c_int32 * MAX_NEWTON_LOG),
                ("n_hvp", C.c_int32), ("hvp_ms", C.c_double), ("ms_phase", C.c_double * 8),
                ("n_cells", C.c_int64), ("n_nodes", C.c_int64), ("n_free_nodes", C.c_int64),
                ("n_launches", C.c_int64), ("grad_norms", C.c_double * MAX_NEWTON_LOG),
                ("alphas", C.c_double * MAX_NEWTON_LOG), ("tangent_format", C.c_int32), ("pad_", C.c_int32)]

    def as_dict(self) -> dict:
        n = min(self.newton_iters, MAX_NEWTON_LOG)
        return dict(newton_iters=self.newton_iters, cg_total=self.cg_iters_total, ls_halvings=self.ls_halvings,
                    converged=self.converged, neg_curv=self.neg_curvature,
                    n_inverted_trials=self.n_inverted_trials, grad_norm0=self.grad_norm0,
                    grad_norm=self.grad_norm, energy=self.energy, cg_iters=list(self.cg_iters[:n]),
                    ls_iters=list(self.ls_iters[:n]), n_hvp=self.n_hvp, hvp_ms=self.hvp_ms,
                    ms_phase=list(self.ms_phase), n_cells=self.n_cells, n_nodes=self.n_nodes,
                    n_free_nodes=self.n_free_nodes, n_launches=self.n_launches,
                    grad_norms=list(self.grad_norms[:min(n + 1, MAX_NEWTON_LOG)]), alphas=list(self.alphas[:n]),
                    tangent_format=self.tangent_format)


_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "mpl_create": [_vp, _vp, _vp],
    "mpl_destroy": [_vp],
    "mpl_last_error": [_vp],
    "mpl_set_stream": [_vp, _vp],
    "mpl_version": [],
    "mpl_nccl_unique_id": [_vp],
    "mpl_group_create": [_i32, _vp],
    "mpl_nccl_selftest": [_i32, _vp],
    "mpl_group_destroy": [_vp],
    "mpl_set_slabs": [_vp, _vp],
    "mpl_balance_slabs": [_i32, _vp, _i32, _vp],
    "mpl_set_particle_ids": [_vp, _vp],
    "mpl_get_particle_ids": [_vp, _vp],
    "mpl_get_node_owner": [_vp, _vp],
    "mpl_set_materials": [_vp, _i32, _vp],
    "mpl_set_gravity": [_vp, _vp],
    "mpl_set_dirichlet": [_vp, _i32, _vp],
    "mpl_set_particles": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32],
    "mpl_get_particles": [_vp, _vp, _vp, _vp, _vp, _i32],
    "mpl_num_particles": [_vp],
    "mpl_resample": [_vp, _d, _vp, _vp, _vp],
    "mpl_get_nodes": [_vp, _vp, _vp, _vp, _vp],
    "mpl_get_active_blocks": [_vp, _vp],
    "mpl_get_particle_cells": [_vp, _vp],
    "mpl_get_quadrature": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "mpl_energy": [_vp, _vp, _vp],
    "mpl_gradient": [_vp, _vp, _vp, _vp],
    "mpl_linearize": [_vp, _vp],
    "mpl_get_diag": [_vp, _vp],
    "mpl_set_psd_projection": [_vp, _i32],
    "mpl_hvp": [_vp, _vp, _vp],
    "mpl_hvp_bench": [_vp, _vp, _vp, _i32, _vp],
    "mpl_newton_step": [_vp, _vp, _vp],
    "mpl_get_velocity": [_vp, _vp],
    "mpl_set_velocity": [_vp, _vp],
    "mpl_transfer_to_particles": [_vp, _d],
    "mpl_step": [_vp, _d, _vp, _vp],
    "mpl_explicit_velocity": [_vp],
    "mpl_stage_particles": [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp],
    "mpl_get_particles_async": [_vp, _vp, _vp, _vp, _vp],
    "mpl_stage_wait": [_vp],
    "mpl_explicit_step": [_vp, _d, _vp],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
_lib.mpl_last_error.restype = C.c_char_p
_lib.mpl_version.restype = C.c_char_p
_lib.mpl_num_particles.restype = C.c_int64
_lib.mpl_destroy.restype = None
_lib.mpl_group_destroy.restype = None


def version() -> str:
    return _lib.mpl_version().decode()


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0; broadcast it to the other ranks before creating contexts)."""
    buf = (C.c_uint8 * 128)()
    st = _lib.mpl_nccl_unique_id(buf)
    if st != 0:
        raise MplError(st, "mpl_nccl_unique_id failed (is libnccl.so.2 loadable?)")
    return bytes(buf)


def nccl_selftest(device: int = 0) -> float:
    """One-rank NCCL transport self-test (returns 8.0)."""
    out = C.c_double()
    st = _lib.mpl_nccl_selftest(int(device), C.byref(out))
    if st != 0:
        raise MplError(st, "mpl_nccl_selftest")
    return out.value


def balance_slabs(weight, nranks: int) -> np.ndarray:
    """Slab cuts (nranks + 1 cell-block x indices) balancing a per-plane weight (host-only call)."""
    w = np.ascontiguousarray(weight, dtype=np.int64)
    cuts = np.zeros(nranks + 1, np.int32)
    st = _lib.mpl_balance_slabs(int(w.size), w.ctypes.data, int(nranks), cuts.ctypes.data)
    if st != 0:
        raise MplError(st, "mpl_balance_slabs")
    return cuts


class Group:
    """In-process loopback group: ranks are host threads of this process (tests on one GPU)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        st = _lib.mpl_group_create(int(nranks), C.byref(h))
        if st != 0:
            raise MplError(st, "mpl_group_create")
        self._h = h
        self.nranks = nranks

    def close(self):
        if getattr(self, "_h", None):
            _lib.mpl_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(a) -> Optional[int]:
    """Raw address of a numpy array or torch tensor (must be contiguous)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "numpy buffer must be C-contiguous"
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous(), "tensor must be contiguous"
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")


@dataclasses.dataclass
class Counts:
    n_cells: int
    n_nodes: int
    n_blocks: int


class Context:
    """One simulation context on one GPU (C ABI mpl_ctx)."""

    def __init__(self, n: Sequence[int], dx: float, precision: int = 32, device: int = 0,
                 origin: Sequence[float] = (0.0, 0.0, 0.0), rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None, group: Optional[Group] = None):
        self._idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        cfg = Config(precision=precision, device=device, rank=rank, nranks=nranks,
                     nccl_unique_id=C.cast(self._idbuf, C.c_void_p) if self._idbuf is not None else None,
                     loopback=group._h if group is not None else None)
        self.rank, self.nranks = rank, nranks
        g = Grid()
        for a in range(3):
            g.n[a] = int(n[a])
            g.origin[a] = float(origin[a])
        g.dx = float(dx)
        h = C.c_void_p()
        st = _lib.mpl_create(C.byref(cfg), C.byref(g), C.byref(h))
        if st != 0:
            raise MplError(st, "mpl_create failed")
        self.n = tuple(int(a) for a in n)
        self._h = h
        self.precision = precision
        self.dtype = np.float32 if precision == 32 else np.float64
        self.nmat = 0
        self.counts: Optional[Counts] = None

    # ---------------------------------------------------------------------------------------
    def _chk(self, st: int, what: str):
        if st != 0:
            raise MplError(st, f"{what}: {_lib.mpl_last_error(self._h).decode()}")

    def close(self):
        if getattr(self, "_h", None):
            _lib.mpl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _real(self, a, shape=None):
        if isinstance(a, np.ndarray):
            a = np.ascontiguousarray(a, dtype=self.dtype)
            if shape is not None:
                assert a.size == int(np.prod(shape)), (a.shape, shape)
        return a

    def _nn(self) -> int:
        # before a (successful) resample there are no nodes: the library then reports the call-order error
        return self.counts.n_nodes if self.counts is not None else 0

    def _out(self, shape, out=None):
        if out is not None:
            return out
        return np.zeros(shape, dtype=self.dtype)

    # ---- scene ----------------------------------------------------------------------------
    def set_stream(self, stream_ptr: Optional[int]):
        self._chk(_lib.mpl_set_stream(self._h, stream_ptr), "mpl_set_stream")

    def set_materials(self, materials):
        arr = (Material * len(materials))()
        for k, m in enumerate(materials):
            arr[k].kind, arr[k].E, arr[k].nu, arr[k].rho = int(getattr(m, "kind", 0)), float(m.E), float(m.nu), float(m.rho)
            arr[k].yield_stress = float(getattr(m, "yield_stress", 0.0))
        self._chk(_lib.mpl_set_materials(self._h, len(materials), arr), "mpl_set_materials")
        self.nmat = len(materials)

    def set_gravity(self, g):
        arr = (C.c_double * 3)(*[float(x) for x in g])
        self._chk(_lib.mpl_set_gravity(self._h, arr), "mpl_set_gravity")

    def set_dirichlet(self, boxes):
        arr = (DirichletBox * max(1, len(boxes)))()
        for b, bx in enumerate(boxes):
            for a in range(3):
                arr[b].lo[a], arr[b].hi[a], arr[b].velocity[a] = bx.lo[a], bx.hi[a], bx.velocity[a]
        self._chk(_lib.mpl_set_dirichlet(self._h, len(boxes), arr), "mpl_set_dirichlet")

    def set_particles(self, x, v, F, G, vol, mat):
        n = int(x.shape[0])
        x, v, F, G, vol = (self._real(a) for a in (x, v, F, G, vol))
        if isinstance(mat, np.ndarray):
            mat = np.ascontiguousarray(mat, dtype=np.int32)
        self._keep = (x, v, F, G, vol, mat)
        on_dev = int(hasattr(x, "is_cuda") and x.is_cuda)
        self._chk(_lib.mpl_set_particles(self._h, n, _ptr(x), _ptr(v), _ptr(F), _ptr(G), _ptr(vol), _ptr(mat),
                                         on_dev), "mpl_set_particles")
        self._keep = None
        self.np = n

    def stage_particles(self, x, v, F, G, vol, mat):
        """Asynchronous set_particles (mpl_stage_particles): the arrays (pinned host memory or torch
        tensors) must stay alive and unchanged until stage_wait(); the next resample adopts them."""
        n = int(x.shape[0])
        x, v, F, G, vol = (self._real(a) for a in (x, v, F, G, vol))
        if isinstance(mat, np.ndarray):
            mat = np.ascontiguousarray(mat, dtype=np.int32)
        self._staged_keep = (x, v, F, G, vol, mat)
        self._chk(_lib.mpl_stage_particles(self._h, n, _ptr(x), _ptr(v), _ptr(F), _ptr(G), _ptr(vol), _ptr(mat)),
                  "mpl_stage_particles")
        self.np = n

    def get_particles_async(self, x, v, F, G):
        """Enqueue the readback (input order) into caller-owned host arrays; complete after stage_wait()."""
        self._chk(_lib.mpl_get_particles_async(self._h, _ptr(x), _ptr(v), _ptr(F), _ptr(G)), "mpl_get_particles_async")

    def stage_wait(self):
        self._chk(_lib.mpl_stage_wait(self._h), "mpl_stage_wait")

    def set_slabs(self, cuts):
        c = np.ascontiguousarray(cuts, dtype=np.int32)
        self._chk(_lib.mpl_set_slabs(self._h, c.ctypes.data), "mpl_set_slabs")

    def set_particle_ids(self, ids):
        a = np.ascontiguousarray(ids, dtype=np.int32)
        self._chk(_lib.mpl_set_particle_ids(self._h, a.ctypes.data), "mpl_set_particle_ids")

    def num_particles(self) -> int:
        return int(_lib.mpl_num_particles(self._h))

    def get_particle_ids(self) -> np.ndarray:
        ids = np.zeros(self.num_particles(), np.int32)
        self._chk(_lib.mpl_get_particle_ids(self._h, _ptr(ids)), "mpl_get_particle_ids")
        return ids

    def get_node_owner(self) -> np.ndarray:
        o = np.zeros(self.counts.n_nodes, np.uint8)
        self._chk(_lib.mpl_get_node_owner(self._h, _ptr(o)), "mpl_get_node_owner")
        return o

    def get_particles(self, x=None, v=None, F=None, G=None):
        n = _lib.mpl_num_particles(self._h)
        x = self._out((n, 3), x)
        v = self._out((n, 3), v)
        F = self._out((n, 9), F)
        G = self._out((n, 9), G)
        self._chk(_lib.mpl_get_particles(self._h, _ptr(x), _ptr(v), _ptr(F), _ptr(G), 0), "mpl_get_particles")
        return x, v, F, G

    # ---- resample -------------------------------------------------------------------------
    def resample(self, dt: float) -> Counts:
        nc, nn, nb = C.c_int64(), C.c_int64(), C.c_int64()
        self._chk(_lib.mpl_resample(self._h, float(dt), C.byref(nc), C.byref(nn), C.byref(nb)), "mpl_resample")
        self.counts = Counts(nc.value, nn.value, nb.value)
        return self.counts

    def get_nodes(self):
        n = self.counts.n_nodes
        ijk = np.zeros((n, 3), np.int32)
        m = np.zeros(n, self.dtype)
        vn = np.zeros((n, 3), self.dtype)
        fr = np.zeros(n, np.uint8)
        self._chk(_lib.mpl_get_nodes(self._h, _ptr(ijk), _ptr(m), _ptr(vn), _ptr(fr)), "mpl_get_nodes")
        return ijk, m, vn, fr

    def get_active_blocks(self) -> np.ndarray:
        ids = np.zeros(self.counts.n_blocks, np.int64)
        self._chk(_lib.mpl_get_active_blocks(self._h, _ptr(ids)), "mpl_get_active_blocks")
        return ids

    def get_particle_cells(self) -> np.ndarray:
        b = np.zeros((self.num_particles(), 3), np.int32)
        self._chk(_lib.mpl_get_particle_cells(self._h, _ptr(b)), "mpl_get_particle_cells")
        return b

    def get_quadrature(self) -> dict:
        n, nm = self.counts.n_cells, self.nmat
        out = dict(ijk=np.zeros((n, 3), np.int32), m_c=np.zeros(n, self.dtype), v_c=np.zeros((n, 3), self.dtype),
                   G_c=np.zeros((n, 9), self.dtype), V_ck=np.zeros((nm, n), self.dtype),
                   tau_ck=np.zeros((nm, n, 9), self.dtype), S_ck=np.zeros((nm, n, 9), self.dtype))
        self._chk(_lib.mpl_get_quadrature(self._h, *[_ptr(out[k]) for k in
                                                      ("ijk", "m_c", "v_c", "G_c", "V_ck", "tau_ck", "S_ck")]),
                  "mpl_get_quadrature")
        return out

    # ---- potential ------------------------------------------------------------------------
    def energy(self, v) -> float:
        v = self._real(v)
        e = C.c_double()
        self._chk(_lib.mpl_energy(self._h, _ptr(v), C.byref(e)), "mpl_energy")
        return e.value

    def gradient(self, v, out=None):
        v = self._real(v)
        g = self._out((self._nn(), 3), out)
        e = C.c_double()
        self._chk(_lib.mpl_gradient(self._h, _ptr(v), _ptr(g), C.byref(e)), "mpl_gradient")
        return g, e.value

    def set_psd_projection(self, on: bool):
        """Tangent of mpl_linearize / mpl_hvp / mpl_get_diag: exact (False) or per-cell PSD-projected (True)."""
        self._chk(_lib.mpl_set_psd_projection(self._h, int(bool(on))), "mpl_set_psd_projection")

    def linearize(self, v):
        v = self._real(v)
        self._chk(_lib.mpl_linearize(self._h, _ptr(v)), "mpl_linearize")

    def get_diag(self, out=None):
        d = self._out((self._nn(), 3), out)
        self._chk(_lib.mpl_get_diag(self._h, _ptr(d)), "mpl_get_diag")
        return d

    def hvp(self, u, out=None):
        u = self._real(u)
        h = self._out((self._nn(), 3), out)
        self._chk(_lib.mpl_hvp(self._h, _ptr(u), _ptr(h)), "mpl_hvp")
        return h

    def hvp_bench(self, u, reps: int, out=None) -> float:
        ms = C.c_double()
        self._chk(_lib.mpl_hvp_bench(self._h, _ptr(u), _ptr(out), int(reps), C.byref(ms)), "mpl_hvp_bench")
        return ms.value

    # ---- solve ----------------------------------------------------------------------------
    @staticmethod
    def solver_cfg(s, fixed_newton: int = 0, fixed_cg=None, fixed_ls=None):
        cfg = SolverCfg(newton_max=s.newton_max, cg_max=s.cg_max, newton_rtol=s.eps_newton, cg_rtol=s.eps_cg,
                        armijo_c=s.armijo, ls_max=s.ls_max, ls_slack=getattr(s, "ls_slack", 1e-13),
                        fixed_newton_iters=int(fixed_newton), psd_project=int(bool(getattr(s, "psd", False))))
        keep = []
        if fixed_cg is not None:
            a = np.ascontiguousarray(fixed_cg, dtype=np.int32)
            keep.append(a)
            cfg.fixed_cg_iters = a.ctypes.data
        if fixed_ls is not None:
            a = np.ascontiguousarray(fixed_ls, dtype=np.int32)
            keep.append(a)
            cfg.fixed_ls_halvings = a.ctypes.data
        return cfg, keep

    def newton_step(self, solver, fixed_newton: int = 0, fixed_cg=None, fixed_ls=None) -> dict:
        cfg, keep = self.solver_cfg(solver, fixed_newton, fixed_cg, fixed_ls)
        st = SolveStats()
        self._chk(_lib.mpl_newton_step(self._h, C.byref(cfg), C.byref(st)), "mpl_newton_step")
        del keep
        return st.as_dict()

    def get_velocity(self, out=None):
        v = self._out((self._nn(), 3), out)
        self._chk(_lib.mpl_get_velocity(self._h, _ptr(v)), "mpl_get_velocity")
        return v

    def set_velocity(self, v):
        v = self._real(v)
        self._chk(_lib.mpl_set_velocity(self._h, _ptr(v)), "mpl_set_velocity")

    def transfer_to_particles(self, dt: float):
        self._chk(_lib.mpl_transfer_to_particles(self._h, float(dt)), "mpl_transfer_to_particles")

    def explicit_velocity(self):
        """Explicit update v^{n+1} = v^n + dt (g + f/m) after resample (Eq. explicitforce)."""
        self._chk(_lib.mpl_explicit_velocity(self._h), "mpl_explicit_velocity")

    def explicit_step(self, dt: float) -> dict:
        st = SolveStats()
        self._chk(_lib.mpl_explicit_step(self._h, float(dt), C.byref(st)), "mpl_explicit_step")
        return st.as_dict()

    def step(self, dt: float, solver, fixed_newton: int = 0, fixed_cg=None, fixed_ls=None) -> dict:
        cfg, keep = self.solver_cfg(solver, fixed_newton, fixed_cg, fixed_ls)
        st = SolveStats()
        self._chk(_lib.mpl_step(self._h, float(dt), C.byref(cfg), C.byref(st)), "mpl_step")
        del keep
        self.counts = Counts(st.n_cells, st.n_nodes, self.counts.n_blocks if self.counts else -1)
        return st.as_dict()


def from_scene(scene, device: int = 0, precision: Optional[int] = None) -> Context:
    """Context initialised with a scenes.Scene (materials, gravity, Dirichlet boxes, particles)."""
    ctx = Context(scene.n, scene.dx, precision or scene.precision, device, scene.origin)
    ctx.set_materials(scene.materials)
    ctx.set_gravity(scene.gravity)
    ctx.set_dirichlet(scene.dirichlet)
    ctx.set_particles(scene.x, scene.v, scene.F, scene.G, scene.vol, scene.mat)
    return ctx


def slab_cuts(scene, nranks: int) -> np.ndarray:
    """Cuts balancing the scene's particles over nranks x-slabs of 4-cell blocks."""
    from .dist import plane_weights
    return balance_slabs(plane_weights(scene.x[:, 0], scene.n[0], scene.dx, scene.origin[0]), nranks)


def slab_select(scene, cuts, rank: int) -> np.ndarray:
    """Indices of the particles rank owns: base cell x-block in [cuts[rank], cuts[rank+1])."""
    bx = np.floor((np.asarray(scene.x[:, 0], np.float64) - scene.origin[0]) / scene.dx - 0.5).astype(np.int64) // 4
    return np.nonzero((bx >= cuts[rank]) & (bx < cuts[rank + 1]))[0]


def from_scene_rank(scene, rank: int, nranks: int, cuts, device: int = 0, precision: Optional[int] = None,
                    nccl_id: Optional[bytes] = None, group: Optional[Group] = None) -> Context:
    """Slab rank `rank` of `nranks`: its owned particles (global ids = scene indices)."""
    ctx = Context(scene.n, scene.dx, precision or scene.precision, device, scene.origin, rank=rank, nranks=nranks,
                  nccl_id=nccl_id, group=group)
    ctx.set_slabs(cuts)
    ctx.set_materials(scene.materials)
    ctx.set_gravity(scene.gravity)
    ctx.set_dirichlet(scene.dirichlet)
    sel = slab_select(scene, cuts, rank)
    ctx.set_particles(scene.x[sel], scene.v[sel], scene.F[sel], scene.G[sel], scene.vol[sel], scene.mat[sel])
    ctx.set_particle_ids(sel.astype(np.int32))
    return ctx
