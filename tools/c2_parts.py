"""C2 (2D SO8) step time of the cooperative kernel with parts switched off
(FDW_DEBUG_FUSED bit0: no sweep, bit1: no receivers) -- development helper."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model
w = configs.build_workload(configs.CONFIGS[os.environ.get("WL", "C2")](), np.float32)
s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
s.advance_raw(100, record=True)
best = 1e9
for _ in range(3):
    s.reset_state()
    t = time.perf_counter(); s.advance_raw(1500, record=os.environ.get("RECORD", "1") == "1"); best = min(best, time.perf_counter() - t)
print(json.dumps(dict(dbg=os.environ.get("FDW_DEBUG_FUSED", "0"), us_per_step=round(best / 1500 * 1e6, 2),
                      gpts=round(w.grid.extended_points() * 1500 / best / 1e9, 1), layout=s.layout())), flush=True)
