"""Pins the oracle and the host setup mirror to fixtures produced by the
reference itself (oracle/gen_golden.py through oracle/_ref)."""
import numpy as np
import pytest

from helpers import golden_names, load_golden, oracle_solver, same, sha
from paper_2201_05278_b200.configs import build_workload


@pytest.mark.parametrize("name", golden_names())
def test_host_setup_matches_reference(name):
    cfg, dtype, meta, _, _ = load_golden(name)
    w = build_workload(cfg, dtype)
    assert w.axis.n_steps == meta["n_steps"]
    assert w.axis.dt == meta["dt"]
    assert sha(w.velocity) == meta["sha_velocity"]
    assert sha(w.eta) == meta["sha_eta"]
    assert sha(w.sources.offsets, w.sources.index, w.sources.weight) == meta["sha_sources"]
    assert sha(w.receivers.offsets, w.receivers.index, w.receivers.weight) == meta["sha_receivers"]
    assert sha(w.wavelet) == meta["sha_wavelet"]


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_fixture(name):
    cfg, dtype, meta, seis, final = load_golden(name)
    w = build_workload(cfg, dtype)
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    res = o.forward()
    assert same(res["seismogram"], seis)
    assert same(res["final"], final)
    assert np.abs(final).max() > 0
