"""Strided snapshots streamed by fdw_snapshot_async during an asynchronous
forward (kernel.hpp:237-263, :305-323): every snapshot equals the oracle's
extended level at that step, for pageable and pinned destinations; an
instability inside an asynchronous chunk is reported at the same step."""
import dataclasses

import numpy as np
import pytest

from helpers import D, N, X, gpu_solver, oracle_solver, same, small_config
from paper_2201_05278_b200 import InstabilityError
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu


def _strip(a, h):
    return a[tuple(slice(h, -h) for _ in range(a.ndim))]


def _oracle_snapshots(w, stride):
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    o.refresh_boundary()
    snaps = {0: _strip(np.array(o.current()), w.grid.halo)}
    for n in range(1, w.axis.n_steps + 1):
        assert o.step() is None
        if n % stride == 0:
            snaps[n] = _strip(np.array(o.current()), w.grid.halo)
    return snaps


@pytest.mark.parametrize("ndim,stride", [(2, 1), (2, 7), (3, 5), (3, 16)])
@pytest.mark.parametrize("pinned", [False, True])
def test_streamed_snapshots_match_the_oracle(ndim, stride, pinned):
    shape = (29, 37) if ndim == 2 else (17, 21, 19)
    cfg = small_config(ndim=ndim, order=8, shape=shape, bc=[[N, D], [D, X], [D, N]], steps=40)
    w = build_workload(cfg, np.float32)
    w.axis = dataclasses.replace(w.axis, saving_stride=stride)
    g = gpu_solver(w)
    if pinned:
        import torch

        g.set_host_allocator(lambda shp, dt: torch.empty(shp, dtype=torch.float32).pin_memory().numpy())
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    want = _oracle_snapshots(w, stride)
    assert res.snapshot_steps == sorted(want)
    for step, snap in zip(res.snapshot_steps, res.snapshots):
        assert same(snap, want[step]), step
    assert np.abs(res.snapshots[-1]).max() > 0


def test_instability_inside_an_async_chunk():
    cfg = small_config(ndim=2, order=4, shape=(31, 33), steps=400)
    w = build_workload(cfg, np.float32)
    w.axis = dataclasses.replace(w.axis, dt=w.axis.dt * 3.0, saving_stride=50)
    g = gpu_solver(w)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    assert "unstable" in ref
    with pytest.raises(InstabilityError) as ei:
        g.forward()
    assert ei.value.step() == ref["unstable"][0]
    assert g.step_index() == ref["unstable"][0]
