"""Per-chunk step time across one whole C4 forward (development helper).

Runs the bench's workload from rest in chunks of CHUNK steps (graph-captured,
sources + receivers, health at each chunk end like forward()), timing every
chunk with CUDA events on the library stream, then times each kernel once on
the final (developed) field with profile_steps.  Shows whether the gap between
bench.py's step_ms and sweep_ms comes from the field state along the run.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402

CHUNK = int(os.environ.get("CHUNK", "100"))
w = configs.build_workload(configs.CONFIGS[os.environ.get("WL", "C4")](), np.float32)
st = torch.cuda.Stream()
s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
s.set_stream(st.cuda_stream)
s.set_sources(w.sources, w.wavelet)
s.set_receivers(w.receivers)
n = w.axis.n_steps
s.advance_raw(CHUNK, record=True)  # warm-up (graph capture), then restart
s.reset_state()
torch.cuda.synchronize()
out = []
done = 0
while done < n:
    k = min(CHUNK, n - done)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.advance_raw(k, record=True)
    e1.record(st)
    e1.synchronize()
    out.append(round(e0.elapsed_time(e1) / k * 1000.0, 1))
    done += k
# FORWARDS more whole forwards first (bench.py runs 3 + 5 before its profile)
for _ in range(int(os.environ.get("FORWARDS", "0"))):
    s.reset_state()
    s.refresh_boundary()
    s.advance_raw(n, record=True)
torch.cuda.synchronize()
# after the run: per-launch profiles of different lengths, interleaved with
# graph-captured chunks, all from the developed state
after = []
for kind, m in (("profile", 20), ("chunk", 100), ("profile", 200), ("chunk", 100), ("profile", 20), ("chunk", 100)):
    if kind == "profile":
        after.append([kind, m, round(s.profile_steps(m)[0] * 1000.0, 1)])
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.advance_raw(m, record=True)
        e1.record(st)
        e1.synchronize()
        after.append([kind, m, round(e0.elapsed_time(e1) / m * 1000.0, 1)])
print(json.dumps({"workload": os.environ.get("WL", "C4"), "chunk": CHUNK, "us_per_step": out,
                  "mean_us": round(sum(out) / len(out), 1),
                  "after_run_us": after}))
