"""bench.py's e2e loop with per-phase timers (C4)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2201_05278_b200 import configs, Solver, make_material_model, DampingField

w = configs.build_workload(configs.overthrust3d(8), np.float32)
stream = torch.cuda.Stream()
vel = torch.from_numpy(w.velocity).pin_memory().numpy()
eta = torch.from_numpy(w.eta).pin_memory().numpy()
mats = make_material_model(vel)
pinned = {}
def alloc(shape, dtype):
    key = (tuple(shape), np.dtype(dtype).str)
    if key not in pinned:
        pinned[key] = torch.empty(shape, dtype=torch.from_numpy(np.zeros(0, dtype)).dtype).pin_memory().numpy()
    return pinned[key]
use_stream = "nostream" not in sys.argv
for it in range(4):
    T = []
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = Solver(w.grid, mats, DampingField(eta=eta), w.spec, w.axis, w.coeffs)
    T.append(("ctor", time.perf_counter() - t0)); t = time.perf_counter()
    if use_stream:
        s.set_stream(stream.cuda_stream)
    T.append(("set_stream", time.perf_counter() - t)); t = time.perf_counter()
    s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
    T.append(("maps", time.perf_counter() - t)); t = time.perf_counter()
    s.set_host_allocator(alloc)
    r = s.forward()
    T.append(("forward", time.perf_counter() - t)); T.append(("kernel_seconds", r.kernel_seconds)); t = time.perf_counter()
    s.close()
    torch.cuda.synchronize()
    T.append(("close", time.perf_counter() - t))
    print(it, f"total {time.perf_counter()-t0:.3f}", " ".join(f"{k}={v*1e3:.1f}" for k, v in T), flush=True)
