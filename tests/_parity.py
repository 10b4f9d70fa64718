"""Helpers shared by the GPU parity tests: run the oracle and the CUDA path (through the C ABI) on
the same seeded scene and line their outputs up by (i,j,k) key."""
import numpy as np

import oracle


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm((a - b).ravel())
    n = np.linalg.norm(b.ravel())
    return float(d / n) if n > 0 else float(d)


TOL = {64: dict(grad=1e-10, hvp=1e-10, unload=1e-10, step=1e-8),
       32: dict(grad=1e-5, hvp=1e-5, unload=1e-5, step=1e-4)}


def node_ids(grid: oracle.Grid, ijk: np.ndarray) -> np.ndarray:
    n1, n2 = int(grid.n[1]) + 1, int(grid.n[2]) + 1
    return (ijk[:, 0].astype(np.int64) * n1 + ijk[:, 1]) * n2 + ijk[:, 2]


def cell_ids(grid: oracle.Grid, ijk: np.ndarray) -> np.ndarray:
    n1, n2 = int(grid.n[1]), int(grid.n[2])
    return (ijk[:, 0].astype(np.int64) * n1 + ijk[:, 1]) * n2 + ijk[:, 2]


def gpu_context(scene, precision=None):
    from paper_2602_07853_b200 import mpl
    return mpl.from_scene(scene, 0, precision)


class Pair:
    """Oracle + GPU state for one scene after the unload (resample) phase."""

    def __init__(self, scene):
        self.scene = scene
        self.grid = oracle.Grid(scene.n, scene.dx, scene.origin)
        self.un, self.S, self.prob, self.v0 = oracle.prepare(scene, self.grid)
        self.ctx = gpu_context(scene)
        self.counts = self.ctx.resample(scene.dt)
        self.ijk, self.m, self.vn, self.free = self.ctx.get_nodes()
        self.nid = node_ids(self.grid, self.ijk)

    def to_gpu(self, dense3: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(dense3.reshape(-1, 3)[self.nid], dtype=self.ctx.dtype)

    def to_dense(self, canon3: np.ndarray) -> np.ndarray:
        out = np.zeros((self.grid.nnodes, 3))
        out[self.nid] = canon3
        return out
