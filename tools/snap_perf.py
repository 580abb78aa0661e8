"""Strided-snapshot forward: streamed (fdw_snapshot_async, the forward() path)
vs the synchronous advance + fdw_get_extended loop, on C2 (2D) and C4 (3D)."""
import dataclasses, faulthandler, json, os, sys, time
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2201_05278_b200 import configs, Solver, make_material_model, DampingField
from paper_2201_05278_b200._lib import lib, ptr

def run(name, cfg, stride, reps=3):
    w = configs.build_workload(cfg, np.float32)
    w.axis = dataclasses.replace(w.axis, saving_stride=stride)
    s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
    s.set_snapshot_cap(1 << 40)
    s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
    ext = tuple(w.grid.extended_shape[:w.grid.ndim])
    n_snap = w.axis.snapshot_count()
    pinned = [torch.empty(ext, dtype=torch.float32).pin_memory().numpy() for _ in range(n_snap + 1)]
    it = iter(range(10**9))
    out = {}
    for mode in ("stream_pageable", "stream_pinned", "sync_pageable"):
        print("mode", name, stride, mode, file=sys.stderr, flush=True)
        ts = []
        for r in range(reps + 1):
            s.reset_state()
            if mode == "stream_pinned":
                k = iter(range(len(pinned)))
                s.set_host_allocator(lambda shp, dt: pinned[next(k)] if tuple(shp) == ext else np.empty(shp, dt))
            else:
                s.set_host_allocator(None)
            t0 = time.perf_counter()
            if mode.startswith("stream"):
                res = s.forward()
            else:  # the pre-streaming loop: synchronous advance + download per stride
                s.refresh_boundary(); lib().fdw_record(s.ctx)
                snaps = []
                for _ in range(w.axis.n_steps // stride):
                    s.advance_raw(stride, record=True)
                    o = np.empty(ext, np.float32); lib().fdw_get_extended(s.ctx, ptr(o)); snaps.append(o)
                rem = w.axis.n_steps % stride
                if rem: s.advance_raw(rem, record=True)
                lib().fdw_synchronize(s.ctx)
            el = time.perf_counter() - t0
            if r: ts.append(el)
        out[mode] = round(min(ts), 4)
    pts = w.grid.extended_points() * w.axis.n_steps
    print(json.dumps({"case": name, "stride": stride, "snapshots": n_snap, "seconds": out,
                      "gpts": {k: round(pts / v / 1e9, 2) for k, v in out.items()}}), flush=True)

run("C2", configs.marmousi2d(8), 10)
run("C2", configs.marmousi2d(8), 100)
run("C4", configs.overthrust3d(8), 265, reps=2)
