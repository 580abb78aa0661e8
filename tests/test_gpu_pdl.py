"""Programmatic dependent launch (PDL) changes only WHEN kernels start, never
what they compute: the TMA sweep and the point-source kernel prefetch their
setup-time data before griddepcontrol.wait.  The same runs with FDW_NO_PDL=1
(read when the Solver is created) must give bit-identical seismograms and final
levels -- point sources and receivers, constant and variable density, the
CUDA-graph chunks (>= 8 steps) and the direct-launch path (< 8 steps)."""
import os

import numpy as np
import pytest

from helpers import gpu_solver, same, small_config
from paper_2201_05278_b200 import make_material_model
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu


def _run(w, rho, no_pdl):
    if no_pdl:
        os.environ["FDW_NO_PDL"] = "1"
    else:
        os.environ.pop("FDW_NO_PDL", None)
    try:
        from paper_2201_05278_b200 import DampingField, Solver
        mats = make_material_model(w.velocity, rho) if rho is not None else make_material_model(w.velocity)
        s = Solver(w.grid, mats, DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
        assert s.layout()["variant"] == 3
        s.set_sources(w.sources, w.wavelet)
        s.set_receivers(w.receivers)
        res = s.forward()
        out = np.asarray(res.seismogram.data).copy(), res.snapshots[-1].copy()
        s.close()
        return out
    finally:
        os.environ.pop("FDW_NO_PDL", None)


@pytest.mark.parametrize("steps", [5, 130], ids=["direct", "graph"])
@pytest.mark.parametrize("density", [False, True], ids=["const", "vd"])
def test_pdl_on_off_bit_identical(steps, density):
    cfg = small_config(ndim=3, order=8, shape=(29, 33, 37), steps=steps, n_rec=15)
    w = build_workload(cfg, np.float32)
    rho = None
    if density:
        z = np.arange(w.velocity.shape[0], dtype=np.float32)[:, None, None]
        rho = np.ascontiguousarray(np.broadcast_to(1000.0 + 3.0 * z, w.velocity.shape), np.float32)
    seis_a, fin_a = _run(w, rho, no_pdl=False)
    seis_b, fin_b = _run(w, rho, no_pdl=True)
    assert np.abs(fin_a).max() > 0
    assert same(seis_a, seis_b)
    assert same(fin_a, fin_b)
