"""Quick device timing of the C4 / C2 workloads (development helper)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_05278_b200 import configs, Solver, make_material_model, DampingField
from paper_2201_05278_b200._lib import *

_cache = {}
def run(name, cfg, steps, density=False, dtype=np.float32, **kw):
    key = (cfg.name, np.dtype(dtype).str)
    if key not in _cache:
        _cache.clear()
        _cache[key] = configs.build_workload(cfg, dtype)
    w = _cache[key]
    rho = None
    if density:  # layered density (g/cm^3) following the velocity, Gardner-like
        rho = (0.31 * np.power(w.velocity.astype(np.float64), 0.25)).astype(w.velocity.dtype)
    s = Solver(w.grid, make_material_model(w.velocity, rho), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs, **kw)
    s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
    s.advance_raw(100, record=True)  # warm (graph capture)
    pts = w.grid.extended_points()
    t = time.time(); s.advance_raw(steps, record=True); el = time.time() - t
    ms = s.profile_steps(20)
    out = dict(name=name, kw={k: int(v) for k, v in kw.items()}, layout=s.layout(),
               gpts=round(pts * steps / el / 1e9, 2), ms_step=round(el / steps * 1e3, 4), prof_ms=[round(x, 4) for x in ms],
               sweep_gbs=round(pts * 5 * np.dtype(dtype).itemsize / (ms[0] * 1e-3) / 1e9, 1))
    print(json.dumps(out), flush=True)
    s.close()

if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    c4 = configs.overthrust3d(8)
    if "zsweep" in which:
        for zs in (4, 5, 6, 7, 8, 9, 10, 12, 14):
            run(f"C4-zseg{zs}", c4, 200, z_segments=zs)
        c3 = configs.overthrust3d(4)
        for zs in (4, 6, 8, 10):
            run(f"C3-zseg{zs}", c3, 200, z_segments=zs)
        sys.exit(0)
    if "c4only" in which:
        run("C4-tma", c4, 400)
        run("C4-tma-fma", c4, 400, math=FDW_MATH_FMA)
        sys.exit(0)
    if "f64" in which:
        run("C4-f64", c4, 400, dtype=np.float64)
        run("C4-f32", c4, 400)
        run("C2-f64", configs.marmousi2d(8), 1600, dtype=np.float64)
        run("C4-vd-f64", c4, 200, density=True, dtype=np.float64)
        sys.exit(0)
    if "vd" in which:
        run("C4-vd", c4, 200, density=True)
        run("C2-vd", configs.marmousi2d(8), 1600, density=True)
        sys.exit(0)
    if "2d" in which:
        run("C2", configs.marmousi2d(8), 1600)
        c2 = configs.marmousi2d(8); c2.alpha = 0.0
        run("C2-alpha0", c2, 1600)
        run("C2-simple", configs.marmousi2d(8), 1600, variant=FDW_KERNEL_SIMPLE)
        run("C2-simple-alpha0", c2, 1600, variant=FDW_KERNEL_SIMPLE)
        sys.exit(0)
    run("C4-tma", c4, 400)
    run("C4-zmarch", c4, 400, variant=FDW_KERNEL_ZMARCH)
    run("C4-tma-fma", c4, 400, math=FDW_MATH_FMA)
    for zs in (2, 3, 4, 6, 8):
        run(f"C4-tma-zseg{zs}", c4, 200, z_segments=zs)
    run("C3-tma", configs.overthrust3d(4), 400)
    run("C2", configs.marmousi2d(8), 1600)
    run("C1", configs.marmousi2d(2), 1300)
    run("C2-simple", configs.marmousi2d(8), 1600, variant=FDW_KERNEL_SIMPLE)
