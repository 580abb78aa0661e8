"""Attribution of the C4 step time beyond the sweep, on ONE developed wavefield
in ONE process (development helper; `bench.py` reports step_ms vs sweep_ms).

The field is developed once (DEV steps from rest), downloaded, and every
variant restarts from exactly that state at the same step index, so the power
state (sw_power_cap clocks depend on the data) is the same for all of them.
Variants are interleaved over REPS rounds; each time STEPS graph-captured
steps with CUDA events on the library stream:
  full          sweep + point sources + receivers (side stream) + health
  no_prio       the same with equal launch priorities (FDW_NO_PRIO)
  no_pdl        the same with plain launches (FDW_NO_PDL)
  no_receivers  without receivers
  no_sources    without point sources
  sweep_only    neither
plus the per-kernel event times of profile_steps per variant.  AB="K=V;K=V"
replaces the variant list with full steps that differ in env knobs only.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402

DEV = int(os.environ.get("DEV", "2000"))
N = int(os.environ.get("STEPS", "400"))
REPS = int(os.environ.get("REPS", "3"))
VARIANTS = [("full", 1, 1, {}), ("no_prio", 1, 1, {"FDW_NO_PRIO": "1"}), ("no_pdl", 1, 1, {"FDW_NO_PDL": "1"}),
            ("no_receivers", 1, 0, {}), ("no_sources", 0, 1, {}), ("sweep_only", 0, 0, {})]


def make(w, src, rec, env, stream):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    s.set_stream(stream.cuda_stream)
    if src:
        s.set_sources(w.sources, w.wavelet)
    if rec:
        s.set_receivers(w.receivers)
    return s


def variants():
    """AB="K=V[,K=V];K=V...": full-step variants that differ only in env knobs."""
    ab = os.environ.get("AB")
    if not ab:
        return VARIANTS
    out = []
    for spec in ab.split(";"):
        env = dict(kv.split("=", 1) for kv in spec.split(",") if kv)
        out.append((spec or "default", 1, 1, env))
    return out


def main():
    cfg = configs.CONFIGS[os.environ.get("WL", "C4")]()
    w = configs.build_workload(cfg, np.float32)
    pts = w.grid.extended_points()
    stream = torch.cuda.Stream()
    base = make(w, 1, 1, {}, stream)
    base.advance_raw(DEV, record=True)
    prev, curr = base.previous_level().copy(), base.current_level().copy()
    base.close()
    only = os.environ.get("CASES")
    vs = [v for v in variants() if not only or v[0] in only.split(",")]
    res = {v[0]: [] for v in vs}
    prof_all = {}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(REPS):
        for name, src, rec, env in vs:
            s = make(w, src, rec, env, stream)
            s.previous_level()[...] = prev
            s.current_level()[...] = curr
            s.refresh_boundary()
            s.set_step_index(DEV)
            s._host_view = False  # device state is authoritative from here
            s.advance_raw(100, record=bool(rec))  # capture + warm
            torch.cuda.synchronize()
            ev0.record(stream)
            s.advance_raw(N, record=bool(rec))
            ev1.record(stream)
            torch.cuda.synchronize()
            res[name].append(ev0.elapsed_time(ev1) / N * 1e3)
            if rep == REPS - 1:
                prof_all[name] = [round(x * 1e3, 2) for x in s.profile_steps(50)]
            s.close()
    out = {name: {"us_per_step": round(min(v), 2), "reps": [round(x, 2) for x in v],
                  "gpts": round(pts / min(v) / 1e3, 1)} for name, v in res.items()}
    keys = ["sweep", "inject", "boundary", "receivers", "health", "halo"]
    print(json.dumps({"dev_steps": DEV, "steps": N, "variants": out,
                      "prof_us": {k: dict(zip(keys, v)) for k, v in prof_all.items()}}), flush=True)


if __name__ == "__main__":
    main()
