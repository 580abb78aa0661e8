"""Breaks the e2e (public API, host buffers) forward of C4 into its parts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
from paper_2201_05278_b200 import configs, Solver, make_material_model, DampingField
from paper_2201_05278_b200._lib import lib, ptr

w = configs.build_workload(configs.overthrust3d(8), np.float32)
vel = torch.from_numpy(w.velocity).pin_memory().numpy()
eta = torch.from_numpy(w.eta).pin_memory().numpy()
T = {}
def tic(k, t0): T[k] = T.get(k, 0) + time.perf_counter() - t0
for it in range(3):
    t = time.perf_counter(); mm = make_material_model(vel); tic('material_model', t)
    t = time.perf_counter(); s = Solver(w.grid, mm, DampingField(eta=eta), w.spec, w.axis, w.coeffs); torch.cuda.synchronize(); tic('solver_ctor(create+set_medium)', t)
    t = time.perf_counter(); s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers); tic('maps', t)
    t = time.perf_counter(); s.refresh_boundary(); lib().fdw_record(s.ctx); tic('refresh+record', t)
    t = time.perf_counter(); s.advance_raw(w.axis.n_steps, record=True); tic('advance(2650)', t)
    t = time.perf_counter(); ext = s.extended_level(); tic('snapshot D2H pageable', t)
    pin = torch.empty(ext.shape, dtype=torch.float32).pin_memory().numpy()
    t = time.perf_counter(); lib().fdw_get_extended(s.ctx, ptr(pin)); tic('snapshot D2H pinned', t)
    t = time.perf_counter(); sg = s.seismogram_f64(); tic('seismogram', t)
    t = time.perf_counter(); s.close(); tic('close', t)
for k, v in T.items(): print(f"{k:35s} {v/3*1e3:9.1f} ms")
