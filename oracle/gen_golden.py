"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference headers compiled in place) -- TEST INFRASTRUCTURE ONLY.

Each fixture is a small synthetic run built end to end by the reference's own
setup chain (build_grid -> extend_with_damping -> resample_model ->
make_material_model -> damping_field -> build_time_axis -> build_injection_map
-> ricker_wavelet -> Solver<T>::forward).  Stored: the case parameters, the
seismogram and final extended level, and SHA-256 digests of the setup arrays
(velocity, eta, source/receiver maps, wavelet) so the host mirror's setup can
be pinned without committing megabytes.

Run here (needs /root/reference):  python oracle/gen_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import oracle as O  # noqa: E402
from paper_2201_05278_b200.configs import SyntheticConfig  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
N_, D_, X_ = 1, 0, 2


def cases():
    def c2(name, order, bc, tf, shape=(31, 47)):
        h = 10.0
        return SyntheticConfig(
            name=name, ndim=2, bbox=[0, h * (shape[0] - 1), 0, h * (shape[1] - 1)], spacing=[h, h],
            space_order=order, damping=[0.0, 100.0, 100.0, 100.0], vmin=1500.0, vmax=4700.0, tf=tf,
            sources=[(45.0, 235.0, 0.0)], receivers=[(25.0, 5.0 + 10.0 * k, 0.0) for k in range(40)],
            bc=bc, f0=25.0)

    def c3(name, order, bc, tf, shape=(15, 25, 21)):
        h = 20.0
        return SyntheticConfig(
            name=name, ndim=3, bbox=[0, h * (shape[0] - 1), 0, h * (shape[1] - 1), 0, h * (shape[2] - 1)],
            spacing=[h, h, h], space_order=order, damping=[100.0] * 6, vmin=2000.0, vmax=6000.0, tf=tf,
            sources=[(50.0, 250.0, 210.0)], receivers=[(30.0, 10.0 + 20.0 * k, 210.0) for k in range(22)],
            bc=bc, f0=15.0)

    std = [[N_, D_], [D_, D_], [D_, D_]]
    mix = [[D_, N_], [X_, D_], [N_, X_]]
    return [
        (c2("g2d_so2", 2, std, 0.4), np.float32),
        (c2("g2d_so8", 8, std, 0.4), np.float32),
        (c2("g2d_so8_mix", 8, mix, 0.3), np.float32),
        (c2("g2d_so4_f64", 4, mix, 0.3), np.float64),
        (c3("g3d_so4", 4, std, 0.2), np.float32),
        (c3("g3d_so8", 8, std, 0.2), np.float32),
        (c3("g3d_so8_mix", 8, mix, 0.15), np.float32),
        (c3("g3d_so8_f64", 8, std, 0.1), np.float64),
    ]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    os.makedirs(OUT, exist_ok=True)
    index = {}
    for cfg, dtype in cases():
        run = O.RefRun(cfg, dtype)
        vel, eta = run.fields()
        (so, si, sw), (ro, ri, rw) = run.maps()
        wav = run.wavelet()
        res = run.forward()
        meta = {
            "cfg": {k: (v if not isinstance(v, list) else [list(map(float, x)) if isinstance(x, (list, tuple)) else x
                                                             for x in v])
                    for k, v in cfg.__dict__.items()},
            "dtype": np.dtype(dtype).name, "n_steps": run.n_steps, "dt": run.dt,
            "extended": run.extended, "padded": run.padded,
            "sha_velocity": sha(vel), "sha_eta": sha(eta), "sha_sources": sha(so, si, sw),
            "sha_receivers": sha(ro, ri, rw), "sha_wavelet": sha(wav),
            "generator": "oracle/gen_golden.py via oracle/_ref/libfdwave_ref.so",
        }
        np.savez_compressed(os.path.join(OUT, cfg.name + ".npz"), seismogram=res["seismogram"],
                            final=res["final"], meta=json.dumps(meta))
        index[cfg.name] = {"n_steps": run.n_steps, "dtype": meta["dtype"],
                           "max_abs_final": float(np.abs(res["final"]).max())}
        print(cfg.name, run.n_steps, index[cfg.name]["max_abs_final"])
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
