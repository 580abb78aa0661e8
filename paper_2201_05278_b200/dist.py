"""Multi-GPU host plumbing for the Z-slab decomposition (one process per GPU).

The library owns the data path: the sweep stores the R halo planes straight
into the neighbours' levels over NVLink peer memory and orders the steps with
halo epochs in per-rank sync blocks (fdw_api.cu enqueue_step).  This module only
does the control-plane work around it with torch.distributed:
  * all-gather the peer IPC blobs (link_peers),
  * build each rank's slab workload (configs.build_workload(rank, world)),
  * reduce per-rank partial seismograms in rank order (double) and cast to T,
  * gather halo-stripped slabs for checking.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def link_peers(solver, group=None) -> None:
    """Peer transport (a slab Solver, one process per GPU): all-gather
    every rank's IPC export blob and map the neighbours' levels and all sync
    blocks (fdw_peer_import).  Collective over `group`."""
    import torch.distributed as dist
    blobs = [None] * dist.get_world_size(group)
    dist.all_gather_object(blobs, solver.peer_export(), group=group)
    solver.peer_import(blobs)


def slab_range(n_ext: int, world: int, rank: int) -> tuple:
    b, e = C.c_uint64(), C.c_uint64()
    if _lib.lib().fdw_slab_range(n_ext, world, rank, C.byref(b), C.byref(e)) != 0:
        raise ValueError(f"cannot split {n_ext} planes over {world} ranks")
    return int(b.value), int(e.value)


def reduce_seismogram(partial: np.ndarray, dtype, group=None) -> np.ndarray:
    """Sum of per-rank double partials in rank order (rank 0 first), cast to T.
    For world == 1 this is the reference's own accumulation (acquisition.hpp:
    155-158); for world > 1 the per-receiver sum is split at slab faces."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(partial, np.float64))
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    acc = parts[0].numpy().copy()
    for p in parts[1:]:
        acc += p.numpy()
    return acc.astype(dtype)


def gather_slabs(local_ext: np.ndarray, group=None) -> np.ndarray:
    """Concatenate halo-stripped local slabs along Z (rank order) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(local_ext))
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.shape[0]]), group=group)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return np.concatenate([p[: int(s.item())].numpy() for p, s in zip(parts, sizes)], axis=0)
