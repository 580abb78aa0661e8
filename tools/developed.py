"""C4 solver advanced to a developed wavefield (STEPS, default 2000), then
PROF direct-launch steps (ncu target: the sweeps after the graph steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model

w = configs.build_workload(configs.CONFIGS[os.environ.get("WL", "C4")](), np.float32)
s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
s.set_sources(w.sources, w.wavelet)
s.set_receivers(w.receivers)
s.advance_raw(int(os.environ.get("STEPS", "2000")), record=True)
ms = s.profile_steps(int(os.environ.get("PROF", "20")))
print("profile_steps ms", [round(x, 4) for x in ms])
s.close()
