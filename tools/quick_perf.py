"""Quick device timing of the C4 / C2 workloads (development helper)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_05278_b200 import configs, Solver, make_material_model, DampingField
from paper_2201_05278_b200._lib import *

def run(name, cfg, steps, **kw):
    t = time.time()
    w = configs.build_workload(cfg, np.float32)
    tsetup = time.time() - t
    s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs, **kw)
    s.set_sources(w.sources, w.wavelet); s.set_receivers(w.receivers)
    s.advance_raw(100)  # warm (graph capture)
    pts = w.grid.extended_points()
    t = time.time(); s.advance_raw(steps); el = time.time() - t
    ms = s.profile_steps(20)
    out = dict(name=name, kw={k: int(v) for k, v in kw.items()}, layout=s.layout(), setup_s=round(tsetup, 2),
               gpts=pts * steps / el / 1e9, ms_step=el / steps * 1e3, prof_ms=[round(x, 4) for x in ms],
               sweep_gbs=pts * 20 / (ms[0] * 1e-3) / 1e9)
    print(json.dumps(out), flush=True)
    s.close()

run("C4", configs.overthrust3d(8), 400)
run("C4-simple", configs.overthrust3d(8), 200, variant=FDW_KERNEL_SIMPLE)
run("C4-fma", configs.overthrust3d(8), 400, math=FDW_MATH_FMA)
for zs in (1, 2, 3, 4):
    run(f"C4-zseg{zs}", configs.overthrust3d(8), 200, z_segments=zs)
run("C3", configs.overthrust3d(4), 400)
run("C2", configs.marmousi2d(8), 1600)
run("C1", configs.marmousi2d(2), 1300)
