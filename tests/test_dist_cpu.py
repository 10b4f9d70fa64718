"""The N > 1 path on CPU: two gloo ranks (world_size 2, 127.0.0.1) run the host plumbing of the slab
decomposition (paper_2602_07853_b200/dist.py + the library's host-only mpl_balance_slabs) and check,
with the fp64 oracle standing in for each rank's kernels, the identities the GPU path is built on
(DESIGN.md §6):
  * the ranks agree on the cuts; owned particles partition the scene; ghosts = last cell plane of the
    lower slab;
  * P2Q of a rank's owned cells from its owned + ghost particles equals the global P2Q bit for bit;
  * C2N, gradient, HVP and energy restricted to owned cells (and owner-weighted lumped mass) sum over
    the ranks to the global quantities (the halo sum / allreduce of the GPU path).
The GPU-side transport of the same path is tested on one GPU with the loopback group
(tests/test_gpu_slabs.py)."""
import os
import ctypes
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scene_name):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2602_07853_b200 import dist as pdist
    from paper_2602_07853_b200 import mpl, scenes
    from tests.test_gpu_parity import small_cfg2

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = scenes.cfg1(prestrain=True) if scene_name == "cfg1" else small_cfg2(64)
        # NCCL id handshake (a fixed stand-in id: no GPU / NCCL on this box)
        uid = pdist.share_nccl_id(lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        cuts = pdist.agree_cuts(mpl.slab_cuts(sc, world))
        assert cuts[0] == 0 and cuts[-1] == (sc.n[0] + 3) // 4 and np.all(np.diff(cuts) > 0)
        sel = mpl.slab_select(sc, cuts, rank)
        allsel = [None] * world
        dist.all_gather_object(allsel, sel.tolist())
        cat = np.concatenate([np.asarray(a, np.int64) for a in allsel])
        assert np.array_equal(np.sort(cat), np.arange(sc.n_particles)), "owned particles must partition the scene"
        # balanced: no slab holds more than its share plus one block plane
        w = pdist.plane_weights(sc.x[:, 0], sc.n[0], sc.dx)
        assert max(len(a) for a in allsel) <= sc.n_particles / world + w.max()

        grid = oracle.Grid(sc.n, sc.dx, sc.origin)
        un, S, prob, v0 = oracle.prepare(sc, grid)
        A, B = 4 * int(cuts[rank]), 4 * int(cuts[rank + 1])
        base = oracle.base_cells(grid, sc.x)
        ghost = np.nonzero(base[:, 0] == A - 1)[0]
        assert np.all(pdist.owner_of_plane(cuts, base[ghost, 0] // 4) == rank - 1) if rank > 0 else len(ghost) == 0
        loc = np.sort(np.concatenate([sel, ghost]))
        un_r = oracle.unload(grid, sc.materials, sc.x[loc], sc.v[loc], sc.F[loc], sc.G[loc], sc.vol[loc], sc.mat[loc])
        cx = grid.cell_ijk()[:, 0]
        mine = (cx >= A) & (cx < B)
        assert np.array_equal(un_r.m_c[mine], un.m_c[mine])
        assert np.array_equal(un_r.mv_c[mine], un.mv_c[mine])
        assert np.array_equal(un_r.V_ck[:, mine], un.V_ck[:, mine])
        assert np.array_equal(un_r.Vtau_ck[:, mine], un.Vtau_ck[:, mine])

        # rank-local problem: owned cells only, owner-weighted lumped mass (upper rank owns the cut plane)
        nx = grid.node_ijk()[:, 0]
        own = (nx >= A) & ((nx < B) | (rank == world - 1))
        m_c = np.where(mine, un.m_c, 0.0)
        V_ck = np.where(mine[None, :], un.V_ck, 0.0)
        # C2N partial sums over owned cells -> halo sum -> global nodal mass / momentum
        m_i = np.zeros(grid.nnodes)
        v_i = np.zeros((grid.nnodes, 3))
        oracle.lib().orc_c2n(ctypes.byref(grid.c()),
                             oracle._p(m_c), oracle._p(un.v_c), oracle._p(un.G_c), oracle._p(m_i), oracle._p(v_i))
        mv = m_i[:, None] * v_i
        t = torch.from_numpy(np.concatenate([m_i, mv.ravel()]))
        dist.all_reduce(t)
        t = t.numpy()
        m_sum, mv_sum = t[:grid.nnodes], t[grid.nnodes:].reshape(-1, 3)
        assert np.allclose(m_sum, un.m_i, rtol=1e-14, atol=1e-18)
        act = un.m_i > 0
        assert np.allclose(mv_sum[act] / m_sum[act, None], un.v_i[act], rtol=1e-12, atol=1e-14)

        prob_r = oracle.Problem(grid, sc.materials, sc.dt, un.m_i * own, prob.vhat, prob.freed, m_c, V_ck, S)
        rng = np.random.default_rng(5)
        v = v0 + 0.01 * rng.normal(size=v0.shape) * act[:, None]
        u = np.random.default_rng(4).normal(size=v0.shape) * act[:, None]
        parts = [prob_r.gradient(v).ravel(), prob_r.hvp(v, u).ravel(), prob_r.diag(v).ravel(),
                 np.array([prob_r.energy(v)])]
        t = torch.from_numpy(np.concatenate(parts))
        dist.all_reduce(t)
        t = t.numpy()
        n3 = 3 * grid.nnodes
        g_sum, h_sum, d_sum, e_sum = t[:n3], t[n3:2 * n3], t[2 * n3:3 * n3], t[3 * n3]

        def rel(a, b):
            return np.linalg.norm(a - b) / np.linalg.norm(b)

        assert rel(g_sum, prob.gradient(v).ravel()) < 1e-13
        assert rel(h_sum, prob.hvp(v, u).ravel()) < 1e-13
        assert rel(d_sum, prob.diag(v).ravel()) < 1e-13
        assert abs(e_sum - prob.energy(v)) <= 1e-12 * abs(prob.energy(v))
        mx = pdist.reduce_scalars([float(rank), 1.0], "max")
        sm = pdist.reduce_scalars([float(rank), 1.0], "sum")
        assert mx == [world - 1.0, 1.0] and sm == [world * (world - 1) / 2.0, float(world)]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scene_name", ["cfg1", "cfg2s"])
def test_two_gloo_ranks(scene_name):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), scene_name), nprocs=2, join=True)
