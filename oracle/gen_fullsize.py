"""Full-length 3D parity fixtures from the REFERENCE itself -- TEST INFRASTRUCTURE ONLY.

Runs BASELINE.json's C3 (Overthrust SO4, 2400 steps) and C4 (SO8, 2650 steps)
through oracle/_ref/libfdwave_ref.so -- the reference's own setup chain and
`Solver<float>::forward` (/root/reference/proj/include/fdwave/kernel.hpp:237-263)
compiled in place -- over the WHOLE time axis, on all host cores, and stores:

  seismogram   the full (n_steps+1) x 800 receiver record (float32),
  sha_final    SHA-256 of the final extended level (570 MB at C4, not committed),
  planes       decimated Z planes of the final level (every 4th X/Y node of
               planes z = 5, 30, 108, 200) for a tolerance check when bits differ,
  plane_norms  per-Z-plane sum of squares of the final level (double),
  seconds      the reference's own kernel_seconds for the whole run, with the
               host's core count -- the full-length CPU baseline.

Run here (needs /root/reference; ~20-30 min per case on 8 cores):
    python oracle/gen_fullsize.py [C3] [C4]
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import oracle as O  # noqa: E402
from paper_2201_05278_b200 import configs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
PLANES = (5, 30, 108, 200)
DECIM = 4


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(name: str) -> None:
    cfg = configs.CONFIGS[name]()
    t0 = time.time()
    r = O.RefRun(cfg, np.float32)
    res = r.forward()
    wall = time.time() - t0
    if "unstable" in res:
        raise RuntimeError(f"{name}: reference unstable {res['unstable']}")
    fin = res["final"]
    seis = res["seismogram"].reshape(r.n_steps + 1, r.n_rec)
    meta = {
        "config": name, "cfg": cfg.describe(), "n_steps": r.n_steps, "dt": r.dt, "extended": r.extended,
        "n_rec": r.n_rec, "sha_final": hashlib.sha256(np.ascontiguousarray(fin).tobytes()).hexdigest(),
        "sha_seismogram": hashlib.sha256(np.ascontiguousarray(seis).tobytes()).hexdigest(),
        "planes": list(PLANES), "decim": DECIM,
        "seconds": res["seconds"], "wall_seconds": wall, "threads": os.cpu_count(), "cpu": cpu_model(),
        "gpts_per_s": r.extended[0] * r.extended[1] * r.extended[2] * r.n_steps / res["seconds"] / 1e9,
        "generator": "oracle/gen_fullsize.py via oracle/_ref/libfdwave_ref.so (Solver<float>, Backend::Parallel)",
    }
    planes = np.stack([fin[z, ::DECIM, ::DECIM] for z in PLANES])
    norms = np.einsum("zxy,zxy->z", fin.astype(np.float64), fin.astype(np.float64))
    np.savez_compressed(os.path.join(OUT, f"full_{name.lower()}.npz"), seismogram=seis, planes=planes,
                        plane_norms=norms, meta=json.dumps(meta))
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["C3", "C4"]):
        run(n)
