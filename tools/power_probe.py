"""Step time on a developed C4 wavefield, with nvidia-smi clocks/power sampled
during each timed window (development helper: is the sweep power-capped?).

For each case: advance DEV steps from rest (the wavefield fills the grid),
then time T more graph steps while sampling clocks.
"""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402
from paper_2201_05278_b200._lib import FDW_MATH_EXACT, FDW_MATH_FMA  # noqa: E402

DEV = int(os.environ.get("DEV", "1500"))
T = int(os.environ.get("T", "1000"))


def sample(stop_after):
    return subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                             "-lms", "100"], stdout=subprocess.PIPE, text=True)


def main():
    w = configs.build_workload(configs.CONFIGS[os.environ.get("WL", "C4")](), np.float32)
    pts = w.grid.extended_points()
    cases = [("exact", FDW_MATH_EXACT, 1), ("fma", FDW_MATH_FMA, 1), ("exact_zero", FDW_MATH_EXACT, 0)]
    only = os.environ.get("CASES")
    for name, math, src in cases:
        if only and name not in only.split(","):
            continue
        s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
                   math=math)
        if src:
            s.set_sources(w.sources, w.wavelet)
        s.set_receivers(w.receivers)
        s.advance_raw(DEV, record=True)
        p = sample(0)
        time.sleep(0.3)
        t = time.perf_counter()
        s.advance_raw(T, record=True)
        el = time.perf_counter() - t
        p.terminate()
        out, _ = p.communicate()
        rows = [tuple(float(x) for x in l.split(",")) for l in out.strip().splitlines() if l.strip()]
        rows = rows[3:-1] if len(rows) > 5 else rows
        mhz = sorted(r[0] for r in rows)
        pw = sorted(r[1] for r in rows)
        ms = s.profile_steps(20)
        print(json.dumps(dict(case=name, us_per_step=round(el / T * 1e6, 2), gpts=round(pts * T / el / 1e9, 1),
                              sm_mhz_med=mhz[len(mhz) // 2] if mhz else None,
                              power_med=pw[len(pw) // 2] if pw else None, n=len(rows),
                              prof_sweep_us=round(ms[0] * 1e3, 1))), flush=True)
        s.close()


if __name__ == "__main__":
    main()
