import os, sys, json, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model
N = 400
stream = torch.cuda.Stream()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(s):
    s.set_stream(stream.cuda_stream)
    rng = np.random.default_rng(5)
    s.previous_level()[...] = rng.standard_normal(s.previous_level().shape).astype(np.float32) * 1e-3
    s.current_level()[...] = rng.standard_normal(s.current_level().shape).astype(np.float32) * 1e-3
    s.refresh_boundary(); s._host_view = False
    s.advance_raw(100); torch.cuda.synchronize()
    ev0.record(stream); s.advance_raw(N); ev1.record(stream); torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / N * 1e3
c4 = configs.overthrust3d(8)
w1 = configs.build_workload(c4, np.float32)
s = Solver(w1.grid, make_material_model(w1.velocity), DampingField(eta=w1.eta), w1.spec, w1.axis, w1.coeffs)
full = t(s); lay = s.layout(); s.close()
out = {"C4_one_gpu_us": round(full, 2), "layout": lay}
for P in (2, 4, 8):
    w = configs.build_workload(c4, np.float32, rank=1, world=P)
    zs = [int(x) for x in os.environ.get("ZS", "0").split(",")]
    for z in zs:
        s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs, slab=w.slab, z_segments=z)
        s.peer_loopback()
        us = t(s); l = s.layout(); s.close()
        out[f"P{P}_zseg{l['z_segments']}"] = {"us": round(us, 2), "planes": w.slab[3] - w.slab[2], "eff_vs_ideal": round(full / P / us, 3)}
print(json.dumps(out))
