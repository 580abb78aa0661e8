"""The device-ordered multi-GPU step path (separate GPUs: CUDA-graph chunks,
programmatic dependent launch, boundary CTAs waiting in-kernel for the
neighbours' halo epoch, the last one publishing, the health reduction through
the sync blocks) on ONE GPU, with emulated neighbours (fdw_peer_loopback: their
epochs and health posts are pre-satisfied, the halo planes land in scratch).
Host-ordered groups (test_gpu_peer.py) cover the data path; this covers the
ordering code of a real multi-GPU run: it must run chunk after chunk (health
checks included) without a wait timing out, and report the same step count."""
import numpy as np
import pytest

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rank", [0, 1, 2])
def test_loopback_rank_steps_through_graph_chunks(rank):
    cfg = configs.overthrust3d(8, z_planes_ext=3 * 40)
    cfg.fixed_steps = 250
    w = build_workload(cfg, np.float32, rank=rank, world=3)
    s = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
               slab=w.slab)
    s.peer_loopback()
    s.set_sources(w.sources, w.wavelet)
    s.set_receivers(w.receivers)
    s.refresh_boundary()
    s.advance_raw(250, record=True)  # 100-step graph chunks + tail, health at 100, 200, 250
    assert s.step_index() == 250
    m = s.max_abs()
    assert np.isfinite(m)
    s.close()
