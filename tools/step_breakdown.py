"""Where the C4 step time goes (development helper).

Times 400 graph-captured steps of C4 with pieces of the step removed:
full (sweep + inject + receivers on the side stream + health), no receivers,
no sources, sweep only; plus the per-kernel event times of profile_steps.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402

N = int(os.environ.get("STEPS", "400"))


def main():
    cfg = configs.CONFIGS[os.environ.get("WL", "C4")]()
    w = configs.build_workload(cfg, np.float32)
    pts = w.grid.extended_points()
    cases = (("full", 1, 1), ("no_receivers", 1, 0), ("no_sources", 0, 1), ("sweep_only", 0, 0))
    only = os.environ.get("CASES")
    for name, src, rec in cases:
        if only and name not in only.split(","):
            continue
        s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
        if src:
            s.set_sources(w.sources, w.wavelet)
        if rec:
            s.set_receivers(w.receivers)
        s.advance_raw(100, record=bool(rec))
        best, reps = 1e9, []
        for _ in range(int(os.environ.get("REPS", "3"))):
            s.reset_state()
            t = time.perf_counter()
            s.advance_raw(N, record=bool(rec))
            reps.append(round((time.perf_counter() - t) / N * 1e6, 1))
            best = min(best, time.perf_counter() - t)
        ms = s.profile_steps(20)
        print(json.dumps(dict(case=name, us_per_step=round(best / N * 1e6, 2),
                              gpts=round(pts * N / best / 1e9, 1), reps=reps,
                              prof_us=[round(x * 1e3, 2) for x in ms])), flush=True)
        s.close()


if __name__ == "__main__":
    main()
