"""Multi-GPU host plumbing for the Z-slab decomposition (one process per GPU).

The library owns the data path: the sweep stores the R halo planes straight
into the neighbours' levels over NVLink peer memory and orders the steps with
halo epochs in per-rank sync blocks (fdw_api.cu enqueue_step).  This module only
does the control-plane work around it with torch.distributed:
  * all-gather the peer IPC blobs (link_peers),
  * build each rank's slab workload (configs.build_workload(rank, world)),
  * merge per-rank seismograms exactly (partials + straddling receivers'
    per-tap products in entry order) and cast to T,
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


def split_products(solver, rows: int):
    """This rank's per-tap products of the receivers that straddle a slab face
    (fdw_receiver_split_info / fdw_download_receiver_products): (receiver,
    entry position, products[rows, slots])."""
    L = _lib.lib()
    n = C.c_uint64()
    L.fdw_receiver_split_info(solver.ctx, C.byref(n), None, None)
    m = int(n.value)
    rec = np.zeros(max(m, 1), np.uint64)
    ent = np.zeros(max(m, 1), np.uint64)
    prod = np.zeros((rows, max(m, 1)), np.float64)
    if m:
        u64 = C.POINTER(C.c_uint64)
        L.fdw_receiver_split_info(solver.ctx, C.byref(n), rec.ctypes.data_as(u64), ent.ctypes.data_as(u64))
        rc = L.fdw_download_receiver_products(solver.ctx, _lib.ptr(prod), rows)
        if rc != 0:
            raise RuntimeError("fdw_download_receiver_products failed")
    return rec[:m], ent[:m], prod[:, :m]


def merge_seismogram(partials, splits, n_rec: int) -> np.ndarray:
    """The seismogram (rows x receivers, double) of a slab decomposition, bit-
    identical to the reference's single-domain accumulation
    (acquisition.hpp:155-158): receivers inside one slab come from that
    rank's partial sum (the other ranks hold 0 for them); a receiver whose
    taps straddle a face is recomputed from every rank's per-tap products in
    entry order, summed sequentially from +0.0 (np.add.accumulate is a
    left-to-right running sum)."""
    acc = np.asarray(partials[0], np.float64).reshape(-1, n_rec).copy()
    for p in partials[1:]:
        acc += np.asarray(p, np.float64).reshape(-1, n_rec)
    cols = {}
    for r, (rec, ent, prod) in enumerate(splits):
        for j in range(len(rec)):
            cols.setdefault(int(rec[j]), []).append((int(ent[j]), r, j))
    rows = acc.shape[0]
    for p, lst in cols.items():
        lst.sort()
        m = np.zeros((rows, len(lst) + 1), np.float64)
        for k, (_, r, j) in enumerate(lst):
            m[:, k + 1] = splits[r][2][:rows, j]
        acc[:, p] = np.add.accumulate(m, axis=1)[:, -1]
    return acc.reshape(-1)


def reduce_partials(partial: np.ndarray, dtype, group=None) -> np.ndarray:
    """Sum of per-rank double partial sums in rank order (rank 0 first), cast
    to T -- for partials that carry ALL of a rank's taps (the numpy emulation
    of test_slabs_gloo.py).  A library slab Solver keeps the taps of
    receivers that straddle a face as products instead (its partial holds 0
    there): use gather_seismogram for it.  Collective."""
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


def gather_seismogram(solver, dtype, group=None, rows=None) -> np.ndarray:
    """The whole seismogram of a slab decomposition on every rank of `group`,
    cast to T: per-rank partials plus the straddling receivers' per-tap
    products, merged exactly (merge_seismogram).  Collective."""
    import torch.distributed as dist
    rows = solver.time_axis().n_steps + 1 if rows is None else rows
    mine = (solver.seismogram_f64(rows), split_products(solver, rows))
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, mine, group=group)
    return merge_seismogram([p[0] for p in parts], [p[1] for p in parts], solver._n_rec).astype(dtype)


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


reduce_seismogram = gather_seismogram  # the library path: exact at any slab count
