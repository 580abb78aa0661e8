import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_05278_b200 import configs, Solver, make_material_model, DampingField
w = configs.build_workload(configs.marmousi2d(8), np.float32)
s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
s.advance_raw(200, record=True)
print("ok")
