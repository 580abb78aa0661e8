"""Small propagations for compute-sanitizer (racecheck / synccheck / memcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py tma ragged vd 2d peer

Each case runs the production path on a grid small enough for the sanitizer
(seconds, not minutes) and checks the result against the C oracle, so a clean
report is about the same code that the parity tests hold bit-exact:
  tma     3D SO8 TMA sweep, CUDA-graph chunk with programmatic dependent launch
          (sources + receivers), then direct launches
  ragged  3D SO8 with X / Y extents that are not tile multiples and 3 Z segments
  vd      3D SO8 variable density (6 tiles per plane stage)
  2d      2D SO8 shared-memory-resident cooperative kernel (two steps per barrier)
  peer    3 Z slabs on one GPU, host-ordered peer transport (halo stores from
          the sweep, in-kernel epoch waits that find their flags already set)
"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)

from helpers import D, N, X, gpu_solver, oracle_solver, same, small_config  # noqa: E402
from paper_2201_05278_b200 import make_material_model  # noqa: E402
from paper_2201_05278_b200.configs import build_workload  # noqa: E402


def check(w, res, rho=None):
    o = oracle_solver(w) if rho is None else None
    if o is None:
        import oracle as O
        o = O.OracleSolver(w.grid.ndim, w.grid.space_order, w.velocity.dtype, w.grid.extended_shape,
                           w.grid.spacing, w.axis.dt, w.axis.n_steps, w.spec.face, w.velocity, w.eta, density=rho)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    assert same(res.snapshots[-1], ref["final"]), "final level differs from the oracle"
    assert same(np.asarray(res.seismogram.data), ref["seismogram"]), "seismogram differs from the oracle"


def run(cfg, rho=None, **kw):
    w = build_workload(cfg, np.float32)
    from paper_2201_05278_b200 import DampingField, Solver
    mats = make_material_model(w.velocity, rho) if rho is not None else make_material_model(w.velocity)
    s = Solver(w.grid, mats, DampingField(eta=w.eta), w.spec, w.axis, w.coeffs, **kw)
    s.set_sources(w.sources, w.wavelet)
    s.set_receivers(w.receivers)
    res = s.forward()
    check(w, res, rho)
    s.close()


def case_tma():
    run(small_config(ndim=3, order=8, shape=(21, 27, 25), steps=24, n_rec=6))
    run(small_config(ndim=3, order=8, shape=(21, 27, 25), steps=5, n_rec=6))  # direct launches


def case_ragged():
    run(small_config(ndim=3, order=8, shape=(31, 23, 71), steps=12, n_rec=6, bc=[[N, D], [D, X], [N, D]]),
        z_segments=3)


def case_vd():
    cfg = small_config(ndim=3, order=8, shape=(21, 19, 25), steps=12, n_rec=6)
    w = build_workload(cfg, np.float32)
    z = np.arange(w.velocity.shape[0], dtype=np.float32)[:, None, None]
    rho = np.ascontiguousarray(np.broadcast_to(1000.0 + 5.0 * z, w.velocity.shape), np.float32)
    run(cfg, rho=rho)


def case_2d():
    run(small_config(ndim=2, order=8, shape=(61, 97), steps=40, n_rec=20))


def case_peer():
    h = 20.0
    cfg = small_config(ndim=3, order=8, shape=(41, 27, 25), bc=[[N, D], [D, X], [D, N]], n_rec=9,
                       src=[(h * 11.5, h * 13.5, h * 12.5)], steps=16)
    world = 3
    ws = [build_workload(cfg, np.float32, rank=r, world=world) for r in range(world)]
    ss = [gpu_solver(w, slab=w.slab) for w in ws]
    for s, w in zip(ss, ws):
        s.set_sources(w.sources, w.wavelet)
        s.set_receivers(w.receivers)
    for s in ss:
        s.peer_link(ss)
    out, err = [None] * world, []

    def go(r):
        try:
            out[r] = ss[r].forward()
        except Exception as e:  # surfaced below
            err.append(repr(e))

    th = [threading.Thread(target=go, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    full = np.concatenate([o.snapshots[-1] for o in out], axis=0)
    w = build_workload(cfg, np.float32)
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    ref = o.forward()
    assert same(full, ref["final"])
    for s in ss:
        s.close()


CASES = {"tma": case_tma, "ragged": case_ragged, "vd": case_vd, "2d": case_2d, "peer": case_peer}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print(f"case {name} ok", flush=True)
