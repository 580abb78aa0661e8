"""GPU path vs the reference's own outputs (tests/golden), bit for bit."""
import numpy as np
import pytest

from helpers import golden_names, gpu_solver, load_golden, same
from paper_2201_05278_b200._lib import FDW_KERNEL_FUSED2D, FDW_KERNEL_SIMPLE, FDW_KERNEL_TMA, FDW_KERNEL_ZMARCH
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("variant", [FDW_KERNEL_SIMPLE, FDW_KERNEL_ZMARCH, FDW_KERNEL_TMA, FDW_KERNEL_FUSED2D])
def test_gpu_matches_reference_fixture(name, variant):
    cfg, dtype, meta, seis, final = load_golden(name)
    w = build_workload(cfg, dtype)
    g = gpu_solver(w, variant=variant)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    assert same(res.seismogram.data, seis)
    assert same(res.snapshots[-1], final)
