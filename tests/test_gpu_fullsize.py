"""Parity at the BASELINE.json sizes on the production path,
over the WHOLE time axis.

C1/C2 (2D): against the C oracle run in the same job.  C3 (2400 steps) and C4
(2650 steps): against fixtures the REFERENCE itself produced over the full time
axis (oracle/gen_fullsize.py: oracle/_ref/libfdwave_ref.so, the reference's
setup chain and Solver<float>::forward, kernel.hpp:237-263): the whole
receiver seismogram, decimated planes and per-plane energies of the final
level, and SHA-256 digests of both.  The north-star tolerance (relative L2
<= 1e-4 after the full timestep count) is asserted first; EXACT mode must then
match the reference bit for bit (the digests)."""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import gpu_solver, oracle_solver, rel_l2, same
from paper_2201_05278_b200 import configs
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-4  # north star: relative L2 after the full timestep count


@pytest.mark.parametrize("name,make", [("C1", lambda: configs.marmousi2d(2)), ("C2", lambda: configs.marmousi2d(8))],
                         ids=["C1", "C2"])
def test_fullsize_2d_parity(name, make):
    w = build_workload(make(), np.float32)
    g = gpu_solver(w)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    seis = np.asarray(res.seismogram.data)
    assert np.abs(ref["seismogram"]).max() > 0
    assert np.abs(ref["final"]).max() > 0
    assert rel_l2(seis, ref["seismogram"]) <= TOL and rel_l2(res.snapshots[-1], ref["final"]) <= TOL
    assert same(seis, ref["seismogram"]), name
    assert same(res.snapshots[-1], ref["final"]), name


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_fullsize_3d_whole_time_axis_vs_reference(name):
    z = np.load(os.path.join(GOLDEN, f"full_{name.lower()}.npz"))
    meta = json.loads(str(z["meta"]))
    w = build_workload(configs.CONFIGS[name](), np.float32)
    assert w.axis.n_steps == meta["n_steps"] and list(w.grid.extended_shape[:3]) == meta["extended"]
    g = gpu_solver(w)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    seis = np.asarray(res.seismogram.data).reshape(w.axis.n_steps + 1, w.receivers.n_points)
    fin = res.snapshots[-1]
    g.close()
    want = z["seismogram"]
    assert np.abs(want).max() > 0
    # the stated tolerance first (seismogram; decimated final planes; plane energies)
    assert rel_l2(seis, want) <= TOL, rel_l2(seis, want)
    planes = np.stack([fin[p, ::meta["decim"], ::meta["decim"]] for p in meta["planes"]])
    assert rel_l2(planes, z["planes"]) <= TOL
    norms = np.einsum("zxy,zxy->z", fin.astype(np.float64), fin.astype(np.float64))
    assert rel_l2(norms, z["plane_norms"]) <= TOL
    # EXACT mode: the reference's bits over all 2400 / 2650 steps
    assert same(seis, want)
    assert _sha(seis) == meta["sha_seismogram"]
    assert _sha(fin) == meta["sha_final"], f"{name}: final level differs from the reference"
