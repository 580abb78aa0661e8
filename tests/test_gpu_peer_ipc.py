"""Peer transport bootstrap across processes: two processes (gloo for the host
side) each create rank r of a world-2 slab decomposition with the peer
transport, all-gather their fdw_peer_export blobs and map each other's levels
and sync blocks with cudaIpcOpenMemHandle (dist.link_peers).  Both run on the
one GPU of this box, so no step is advanced here (that would make kernels of
two processes wait on each other; the step protocol itself is covered in one
process by test_gpu_peer.py).  Also the refusals: a blob set of the wrong size,
a second import, and a same-process blob."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import gpu_solver, small_config
from paper_2201_05278_b200 import dist as fdist
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = small_config(ndim=3, order=8, shape=(30, 21, 19))
        w = build_workload(cfg, np.float32, rank=rank, world=world)
        s = gpu_solver(w, slab=w.slab)
        blob = s.peer_export()
        assert len(blob) == 512
        errs = []
        try:
            s.peer_import([blob])  # one blob for a world-2 decomposition
        except ValueError as e:
            errs.append(str(e))
        try:
            s.peer_import([blob, blob])  # own-process blob in the peer's slot
        except ValueError as e:
            errs.append(str(e))
        fdist.link_peers(s)  # the real exchange: IPC-maps rank 1 - r
        try:
            fdist.link_peers(s)
        except Exception as e:
            errs.append(str(e))
        dist.barrier()
        s.close()
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


def test_peer_blobs_map_across_processes():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + (os.getpid() % 2000)
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        errs = got[r]
        assert len(errs) == 3, errs
        assert "one blob per rank" in errs[0]
        assert "fdw_peer_link" in errs[1] or "not rank" in errs[1]
        assert "already" in errs[2]
