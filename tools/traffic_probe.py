"""DRAM bytes of the C4 sweep per variant (development helper).

Each variant starts from the same random (non-zero, normal-range) levels and
runs PROF direct-launch steps; run it under
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
        -k regex:sweep3d_tma --csv python tools/traffic_probe.py
and without ncu for the step times.  Variants (VARIANTS=a,b,...):
  base     the shipped sweep
  pd0      single-ring TMA sweep (FDW_TMA_PD=0)
  no_eta   eta all zero (no damping): the eta stream is skipped everywhere
  zseg1    one Z segment (no warm-up planes)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402

PROF = int(os.environ.get("PROF", "2"))


def main():
    w = configs.build_workload(configs.CONFIGS[os.environ.get("WL", "C4")](), np.float32)
    rng = np.random.default_rng(9)
    prev = (rng.standard_normal(w.velocity.shape) * 1e-2).astype(np.float32)
    curr = (rng.standard_normal(w.velocity.shape) * 1e-2).astype(np.float32)
    for name in os.environ.get("VARIANTS", "base,pd0,no_eta,zseg1").split(","):
        env = {"pd0": {"FDW_TMA_PD": "0"}}.get(name, {})
        os.environ.update(env)
        eta = np.zeros_like(w.eta) if name == "no_eta" else w.eta
        s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=eta), w.spec, w.axis, w.coeffs,
                   z_segments=1 if name == "zseg1" else 0)
        for k in env:
            os.environ.pop(k, None)
        s.previous_level()[...] = prev
        s.current_level()[...] = curr
        s.refresh_boundary()
        s._host_view = False
        ms = s.profile_steps(PROF)
        print(name, "layout", s.layout(), "sweep ms", round(ms[0], 4), flush=True)
        s.close()


if __name__ == "__main__":
    main()
