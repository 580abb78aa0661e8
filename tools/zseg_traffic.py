"""DRAM bytes and duration of one C4 sweep per Z-segment count (run under
ncu --metrics; development helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model
w = configs.build_workload(configs.CONFIGS["C4"](), np.float32)
for zs in [int(x) for x in os.environ.get("ZS", "1,2,3,6,10").split(",")]:
    s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs, z_segments=zs)
    s.set_sources(w.sources, w.wavelet)
    ms = s.profile_steps(3)
    print("zseg", zs, "sweep ms", round(ms[0], 4), flush=True)
    s.close()
