"""Process-group plumbing for the slab decomposition (one process per GPU).

torch.distributed carries only host-side setup: broadcasting the library's NCCL unique id from
rank 0, agreeing on the slab cuts and reducing the bench's scalar results.  Every data-path exchange
(interface-node halo sums, PCG / energy allreduces, particle migration) runs inside libmpmlite.so on
its own NCCL communicator.  The functions here work on any backend (gloo on CPU in the tests, nccl on
the GPU box).
"""
from __future__ import annotations

import os
from typing import Callable, Optional, Sequence

import numpy as np


def env() -> tuple:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 without it)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: Optional[bytes], src: int = 0) -> bytes:
    """Broadcast a small byte string from `src` to every rank of the default process group."""
    import torch.distributed as dist
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def share_nccl_id(make_id: Optional[Callable[[], bytes]] = None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id of the library's communicator; all ranks get it."""
    import torch.distributed as dist
    if make_id is None:
        from . import mpl
        make_id = mpl.nccl_unique_id
    uid = make_id() if dist.get_rank() == 0 else None
    uid = broadcast_bytes(uid, 0)
    assert isinstance(uid, bytes) and len(uid) == 128, "NCCL unique id must be 128 bytes"
    return uid


def plane_weights(x: np.ndarray, n0: int, dx: float, origin0: float = 0.0) -> np.ndarray:
    """Particles per 4-cell block plane along x (base cell floor(x/dx - 1/2), block = cell // 4)."""
    nbx = (n0 + 3) // 4
    bx = np.floor((np.asarray(x, np.float64) - origin0) / dx - 0.5).astype(np.int64) // 4
    return np.bincount(np.clip(bx, 0, nbx - 1), minlength=nbx).astype(np.int64)


def agree_cuts(cuts: Sequence[int]) -> np.ndarray:
    """Check that every rank computed the same cuts (they are derived from the same seeded scene)."""
    import torch
    import torch.distributed as dist
    c = torch.tensor(np.asarray(cuts, np.int64))
    lo, hi = c.clone(), c.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    if not torch.equal(lo, hi):
        raise RuntimeError(f"ranks disagree on the slab cuts: {lo.tolist()} vs {hi.tolist()}")
    return np.asarray(cuts, np.int32)


def reduce_scalars(values: Sequence[float], op: str, device=None) -> list:
    """Max or sum of host scalars over ranks (fp64)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(v) for v in t.cpu().tolist()]


def owner_of_plane(cuts: Sequence[int], bx: np.ndarray) -> np.ndarray:
    """Slab rank owning each cell-block plane index bx (cuts[r] <= bx < cuts[r+1])."""
    return np.searchsorted(np.asarray(cuts), np.asarray(bx), side="right") - 1
