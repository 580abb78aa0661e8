"""The slab sweep order used for multi-GPU runs (first/last Z segments, then
the middle ones on a second stream, with the halo exchange in between) run on
one GPU (FDW_FORCE_SPLIT=1): still bit-exact against the oracle, with point
sources in the first, middle and last segments."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

CHILD = r'''
import os, sys
root = os.path.dirname({here!r})
for p in (root, os.path.join(root, "oracle"), {here!r}):
    sys.path.insert(0, p)
import numpy as np
from helpers import D, N, X, gpu_solver, oracle_solver, same, small_config
from paper_2201_05278_b200.configs import build_workload
h = 20.0
shape = (41, 27, 25)
for zsrc in (2.5, 20.5, 38.5):  # first, middle and last of 4 segments
    src = [(h * zsrc, h * 13.5, h * 12.5)]
    cfg = small_config(ndim=3, order=8, shape=shape, bc=[[N, D], [D, X], [D, N]], src=src)
    for dt in (np.float32, np.float64):
        w = build_workload(cfg, dt)
        g = gpu_solver(w, z_segments=4)
        assert g.layout()["variant"] == 3 and g.layout()["z_segments"] == 4
        g.set_sources(w.sources, w.wavelet)
        g.set_receivers(w.receivers)
        res = g.forward()
        o = oracle_solver(w)
        o.set_sources(w.sources, w.wavelet)
        o.set_receivers(w.receivers)
        ref = o.forward()
        assert np.abs(ref["final"]).max() > 0
        assert same(res.seismogram.data, ref["seismogram"]), (zsrc, dt)
        assert same(res.snapshots[-1], ref["final"]), (zsrc, dt)
print("split ok")
'''


def test_split_sweep_order_is_bit_exact():
    env = dict(os.environ, FDW_FORCE_SPLIT="1")
    r = subprocess.run([sys.executable, "-c", CHILD.format(here=HERE)], capture_output=True, text=True, env=env,
                       timeout=900, cwd=os.path.dirname(HERE))
    assert r.returncode == 0 and "split ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
