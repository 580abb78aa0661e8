import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model
w = configs.build_workload(configs.overthrust3d(8), np.float32)
for it in range(3):
    s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
    s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
    torch.cuda.synchronize()
    t = time.perf_counter(); s.advance_raw(100, record=True); t1 = time.perf_counter() - t
    t = time.perf_counter(); s.advance_raw(100, record=True); t2 = time.perf_counter() - t
    t = time.perf_counter(); s.advance_raw(50, record=True); t3 = time.perf_counter() - t
    t = time.perf_counter(); s.advance_raw(50, record=True); t4 = time.perf_counter() - t
    print(f"iter {it}: first 100 {t1*1e3:.1f} ms, second 100 {t2*1e3:.1f} ms, first 50 {t3*1e3:.1f}, second 50 {t4*1e3:.1f}")
    s.close()
