"""Peer transport (Z slabs, no NCCL) on one GPU: world 2, 3 and 4 slabs driven
from one process, one host thread per rank (fdw_peer_link).  Each step's TMA
sweep stores its first / last R planes straight into the neighbours' levels;
its boundary CTAs wait for the neighbours' halo epoch and the last of them
publishes the next one (a separate publish kernel when a point source writes
into the halo planes after the sweep).

All ranks share this box's one GPU, so the library runs the group
HOST-ORDERED (fdw_peer_link sees the shared device): at every cross-rank point
the rank threads meet at a host barrier and order their streams with events,
so when a kernel checks a flag another launch sets, that launch has already
completed -- no kernel ever waits on a concurrently running grid.

The assembled wavefield and the seismogram must be bit-identical to the
single-domain oracle (receivers whose taps straddle a slab face are merged
from the ranks' per-tap products in entry order)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CHILD = r'''
import os, sys, threading
root = os.path.dirname({here!r})
for p in (root, os.path.join(root, "oracle"), {here!r}):
    sys.path.insert(0, p)
import numpy as np
from helpers import D, N, X, gpu_solver, oracle_solver, same, small_config
from paper_2201_05278_b200.configs import build_workload
from paper_2201_05278_b200.dist import merge_seismogram, split_products
h = 20.0
shape = (41, 27, 25)   # extended Z = 51 planes: slabs 26/25 (world 2), 17/17/17 (world 3)
# (world, sources, interior shape, Z segments): taps across the 2-slab face and
# across both faces of 3 slabs (publish after the point-source kernel); 4 thin
# slabs of 13 planes with automatic Z segments and the sources away from every
# face (the sweep's last boundary CTA publishes)
cases = [(2, [(h * 20.5, h * 13.5, h * 12.5)], shape, 3),
         (3, [(h * 11.5, h * 13.5, h * 12.5), (h * 28.5, h * 9.5, h * 10.5)], shape, 3),
         (4, [(h * 1.5, h * 13.5, h * 12.5), (h * 21.5, h * 9.5, h * 10.5)], (42, 27, 25), 0)]
for world, src, shp, zseg in cases:
    cfg = small_config(ndim=3, order=8, shape=shp, bc=[[N, D], [D, X], [D, N]], src=src, n_rec=9)
    for dt in (np.float32, np.float64):
        ws = [build_workload(cfg, dt, rank=r, world=world) for r in range(world)]
        ss = [gpu_solver(w, slab=w.slab, z_segments=zseg) for w in ws]
        for s, w in zip(ss, ws):
            assert s.layout()["variant"] == 3
            s.set_sources(w.sources, w.wavelet)
            s.set_receivers(w.receivers)
        for s in ss:
            s.peer_link(ss)
        out = [None] * world
        err = []
        def run(r):
            try:
                out[r] = ss[r].forward()
            except Exception as e:  # surfaced below
                err.append(repr(e))
        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in th: t.start()
        for t in th: t.join(120)
        assert not err, err
        full = np.concatenate([o.snapshots[-1] for o in out], axis=0)
        rows = ws[0].axis.n_steps + 1
        seis = merge_seismogram([s.seismogram_f64() for s in ss], [split_products(s, rows) for s in ss],
                                ws[0].receivers.n_points)
        w = build_workload(cfg, dt)
        o = oracle_solver(w)
        o.set_sources(w.sources, w.wavelet)
        o.set_receivers(w.receivers)
        ref = o.forward()
        assert np.abs(ref["final"]).max() > 0
        assert same(full, ref["final"]), (world, dt, float(np.abs(full - ref["final"]).max()))
        # straddling receivers merged from per-tap products: the reference's bits
        assert same(seis.astype(dt), np.asarray(ref["seismogram"]).reshape(-1)), (world, dt)
        for s in ss: s.close()
        print("peer ok", world, np.dtype(dt).name, flush=True)
print("peer all ok")
'''


def test_peer_transport_slabs_bit_exact_on_one_gpu():
    r = subprocess.run([sys.executable, "-c", CHILD.format(here=HERE)], capture_output=True, text=True,
                       timeout=900, cwd=os.path.dirname(HERE))
    assert r.returncode == 0 and "peer all ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("peer ok") == 6, r.stdout


CHILD2 = r'''
import os, sys, threading
root = os.path.dirname({here!r})
for p in (root, os.path.join(root, "oracle"), {here!r}):
    sys.path.insert(0, p)
import numpy as np
from helpers import D, N, X, gpu_solver, oracle_solver, same, small_config
from paper_2201_05278_b200 import InstabilityError, ModulatedField
from paper_2201_05278_b200.configs import build_workload

def run_ranks(fn, world):
    out, err = [None] * world, []
    def go(r):
        try:
            out[r] = fn(r)
        except Exception as e:
            out[r] = e
    th = [threading.Thread(target=go, args=(r,)) for r in range(world)]
    for t in th: t.start()
    for t in th: t.join(120)
    return out

# 1. volume sources (the push kernel carries the halo planes after them)
h = 20.0
cfg = small_config(ndim=3, order=8, shape=(31, 21, 19), bc=[[N, D], [D, D], [D, N]], tf=0.05)
w = build_workload(cfg, np.float32)
rng = np.random.default_rng(7)
field = rng.standard_normal(w.velocity.shape).astype(np.float32)
amp = list(np.sin(np.arange(w.axis.n_steps + 1) * 0.3))
world = 2
ws = [build_workload(cfg, np.float32, rank=r, world=world) for r in range(world)]
ss = [gpu_solver(x, slab=x.slab) for x in ws]
for s, x in zip(ss, ws):
    s.set_sources(x.sources, x.wavelet)
    zb, ze = x.slab[2], x.slab[3]
    s.add_volume_source(ModulatedField(field=np.ascontiguousarray(field[zb:ze + 2 * w.grid.halo]), amplitude=amp))
for s in ss:
    s.peer_link(ss)
out = run_ranks(lambda r: ss[r].forward(), world)
assert all(not isinstance(o, Exception) for o in out), out
full = np.concatenate([o.snapshots[-1] for o in out], axis=0)
o = oracle_solver(w)
o.set_sources(w.sources, w.wavelet)
o.add_volume_source(field, amp)
ref = o.forward()
assert np.abs(ref["final"]).max() > 0
assert same(full, ref["final"]), float(np.abs(full - ref["final"]).max())
for s in ss: s.close()
print("peer volume ok", flush=True)

# 2. an instability: every rank stops at the oracle's step (health reduction over the sync blocks)
cfg = small_config(ndim=3, order=2, shape=(23, 15, 15), damping_cells=0, tf=0.5, bc=[[D, D], [D, D], [D, D]])
w = build_workload(cfg, np.float32)
w.axis.dt *= 1.5
w.axis.n_steps = 1000
w.wavelet = np.resize(w.wavelet, 1001)
o = oracle_solver(w)
o.set_sources(w.sources, w.wavelet)
bad = None
for _ in range(1000):
    bad = o.step()
    if bad:
        break
assert bad is not None
ws = []
for r in range(world):
    x = build_workload(cfg, np.float32, rank=r, world=world)
    x.axis.dt, x.axis.n_steps, x.wavelet = w.axis.dt, 1000, w.wavelet
    ws.append(x)
ss = [gpu_solver(x, slab=x.slab) for x in ws]
for s, x in zip(ss, ws):
    s.set_sources(x.sources, x.wavelet)
for s in ss:
    s.peer_link(ss)
out = run_ranks(lambda r: ss[r].advance_raw(1000), world)
for e in out:
    assert isinstance(e, InstabilityError), out
    assert e.step() == bad[0], (e.step(), bad[0])
for s in ss:
    assert s.step_index() == bad[0]
    s.close()
print("peer instability ok", flush=True)
'''


def test_peer_transport_volume_sources_and_instability():
    r = subprocess.run([sys.executable, "-c", CHILD2.format(here=HERE)], capture_output=True, text=True,
                       timeout=900, cwd=os.path.dirname(HERE))
    assert r.returncode == 0 and "peer instability ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
