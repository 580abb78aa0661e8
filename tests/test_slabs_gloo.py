"""Z-slab decomposition on CPU with world_size 2/3 (gloo): the multi-GPU data
flow -- slab ownership, per-rank slab setup, global-face-only Z boundary fill,
R-plane halo exchange, owner-routed injection, rank-ordered seismogram
reduction -- emulated in numpy and held to the single-domain oracle.

The stencil arithmetic here is numpy float32 in the reference association
(elementwise IEEE ops), so the assembled wavefield must be bit-identical to the
oracle's full-grid run; seismograms differ only by the split of each
receiver's double sum at slab faces."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import D, N, X, oracle_solver, small_config
from paper_2201_05278_b200 import dist as fdist
from paper_2201_05278_b200.configs import build_workload


def _sweep(u, out, c2, om, iop, v, ih, h):
    """kernel.hpp:398-420 on the interior of a padded (local) 3D block."""
    nz, nx, ny = (s - 2 * h for s in u.shape)
    c = (slice(h, h + nz), slice(h, h + nx), slice(h, h + ny))
    uc = u[c]
    lz = v[0] * uc
    lx = v[0] * uc
    ly = v[0] * uc
    for j in range(1, h + 1):
        lz = lz + v[j] * (u[h + j:h + j + nz, c[1], c[2]] + u[h - j:h - j + nz, c[1], c[2]])
        lx = lx + v[j] * (u[c[0], h + j:h + j + nx, c[2]] + u[c[0], h - j:h - j + nx, c[2]])
        ly = ly + v[j] * (u[c[0], c[1], h + j:h + j + ny] + u[c[0], c[1], h - j:h - j + ny])
    rhs = lz * ih[0] + lx * ih[1] + ly * ih[2]
    out[c] = (c2[c] * rhs + np.float32(2) * uc - om[c] * out[c]) * iop[c]


def _boundary(f, h, bc, z_lo, z_hi, p_lo, p_hi):
    """apply_boundary (kernel.hpp:67-102) on a slab: the Z phase only on the
    global faces this rank owns, X/Y phases on its own planes."""
    for axis in range(3):
        v = np.moveaxis(f, axis, 0)
        if axis > 0:
            v = np.moveaxis(f[p_lo:p_hi], axis, 0)
        n_ext = v.shape[0] - 2 * h
        for side in range(2):
            if axis == 0 and not (z_lo if side == 0 else z_hi):
                continue
            b = bc[axis][side]
            face = h if side == 0 else h + n_ext - 1
            o = -1 if side == 0 else 1
            if b == D:
                v[face] = 0
            for k in range(1, h + 1):
                v[face + o * k] = -v[face - o * k] if b == D else (v[face - o * k] if b == N else 0)


def _worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = build_workload(cfg, np.float32, rank=rank, world=world)
        g = w.grid
        h = g.halo
        zb, ze = w.slab[2], w.slab[3]
        L = ze - zb + 2 * h
        P1, P2 = g.padded_shape()[1:]
        assert w.velocity.shape == (L, P1, P2)
        dt = w.axis.dt
        c = w.velocity.astype(np.float64)
        edt = w.eta.astype(np.float64) * dt
        c2 = (c * c * dt * dt).astype(np.float32)
        om = (1.0 - edt).astype(np.float32)
        iop = (1.0 / (1.0 + edt)).astype(np.float32)
        v = np.asarray(w.coeffs.second, np.float32)
        ih = [np.float32(1.0 / (sp * sp)) for sp in g.spacing]
        prev = np.zeros((L, P1, P2), np.float32)
        curr = np.zeros((L, P1, P2), np.float32)
        gP12 = P1 * P2
        # owner-routed sources / receivers (global padded flat -> local flat)
        def local(flat):
            gp = int(flat) // gP12
            z = gp - h
            if not (zb <= z < ze):
                return None
            return (gp - zb) * gP12 + int(flat) % gP12
        src = [(local(i), wt) for i, wt in zip(w.sources.index, w.sources.weight)]
        src = [(i, wt) for i, wt in src if i is not None]
        recs = []
        for p in range(w.receivers.n_points):
            a, b = int(w.receivers.offsets[p]), int(w.receivers.offsets[p + 1])
            ent = [(local(i), wt) for i, wt in zip(w.receivers.index[a:b], w.receivers.weight[a:b])]
            recs.append([(i, wt) for i, wt in ent if i is not None])
        z_lo, z_hi = rank == 0, rank == world - 1
        p_lo = 0 if z_lo else h
        p_hi = L if z_hi else L - h
        seis = np.zeros((w.axis.n_steps + 1, len(recs)))

        def exchange(f):
            reqs = []
            import torch
            t = torch.from_numpy(f)
            if rank > 0:
                reqs.append(dist.isend(t[h:2 * h].clone(), rank - 1))
                buf = torch.empty_like(t[0:h])
                dist.recv(buf, rank - 1)
                f[0:h] = buf.numpy()
            if rank < world - 1:
                reqs.append(dist.isend(t[L - 2 * h:L - h].clone(), rank + 1))
                buf = torch.empty_like(t[L - h:L])
                dist.recv(buf, rank + 1)
                f[L - h:L] = buf.numpy()
            for r in reqs:
                r.wait()

        def record(row, f):
            flat = f.reshape(-1)
            for k, ent in enumerate(recs):
                acc = 0.0
                for i, wt in ent:
                    acc += wt * float(flat[i])
                seis[row, k] = acc

        _boundary(curr, h, w.spec.face, z_lo, z_hi, p_lo, p_hi)
        exchange(curr)
        record(0, curr)
        for n in range(w.axis.n_steps):
            _sweep(curr, prev, c2, om, iop, v, ih, h)
            amp = w.wavelet[n]
            pf = prev.reshape(-1)
            for i, wt in src:
                pf[i] += c2.reshape(-1)[i] * np.float32(wt * amp) * iop.reshape(-1)[i]
            prev, curr = curr, prev
            _boundary(curr, h, w.spec.face, z_lo, z_hi, p_lo, p_hi)
            exchange(curr)
            record(n + 1, curr)
        full = fdist.gather_slabs(curr[h:L - h, h:P1 - h, h:P2 - h])
        sg = fdist.reduce_partials(seis, np.float64)
        if rank == 0:
            q.put((full, sg, np.asarray(w.velocity), (zb, ze)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("order", [4, 8])
def test_slab_decomposition_matches_single_domain(world, order):
    cfg = small_config(ndim=3, order=order, shape=(20, 15, 13), damping_cells=3, tf=0.05, n_rec=6,
                       bc=[[N, D], [D, X], [N, D]], src=[(140.0, 150.0, 130.0)])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + 7 * world + order
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    full, sg, _, _ = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = build_workload(cfg, np.float32)
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    assert np.array_equal(full, ref["final"]), "assembled slabs differ from the single-domain run"
    want = ref["seismogram"].reshape(w.axis.n_steps + 1, -1).astype(np.float64)
    assert np.allclose(sg, want, rtol=1e-6, atol=1e-6 * np.abs(want).max())
    assert np.abs(full).max() > 0


@pytest.mark.parametrize("world", [2, 4])
def test_rank_slab_fields_are_slices_of_the_full_fields(world):
    cfg = small_config(ndim=3, order=8, shape=(30, 11, 9), damping_cells=2, tf=0.02)
    full = build_workload(cfg, np.float32)
    h = full.grid.halo
    for r in range(world):
        wr = build_workload(cfg, np.float32, rank=r, world=world)
        zb, ze = wr.slab[2], wr.slab[3]
        assert np.array_equal(wr.velocity, full.velocity[zb:ze + 2 * h])
        assert np.array_equal(wr.eta, full.eta[zb:ze + 2 * h])
