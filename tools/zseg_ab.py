"""Z-segment count of the TMA sweep under the power cap (development helper).
Whole C4 forwards from rest (the bench's step), interleaved over REPS rounds,
for each forced segment count (0 = pick_zseg's choice)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402
from paper_2201_05278_b200._lib import lib  # noqa: E402

SEGS = [int(x) for x in os.environ.get("SEGS", "0,3,4,5,8").split(",")]
REPS = int(os.environ.get("REPS", "2"))
w = configs.build_workload(configs.CONFIGS[os.environ.get("WL", "C4")](), np.float32)
n = w.axis.n_steps
st = torch.cuda.Stream()
res = {z: [] for z in SEGS}
lay = {}
for _ in range(REPS):
    for z in SEGS:
        s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
                   z_segments=z)
        s.set_stream(st.cuda_stream)
        s.set_sources(w.sources, w.wavelet)
        s.set_receivers(w.receivers)
        s.advance_raw(100, record=True)
        s.reset_state()
        s.refresh_boundary()
        lib().fdw_record(s.ctx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.advance_raw(n, record=True)
        e1.record(st)
        e1.synchronize()
        res[z].append(round(e0.elapsed_time(e1) / n * 1000.0, 1))
        lay[z] = s.layout()["z_segments"]
        s.close()
print(json.dumps({"workload": os.environ.get("WL", "C4"), "us_per_step": res, "segments": lay}))
