"""SlabSolver: the Python Solver over several GPUs (one Z slab each), the
counterpart of the C++ drop-in's FDW_DEVICES.  Emulated here with repeated
ordinals on the box's one GPU (host-ordered).  Same public API and results as
the one-domain Solver: forward() field bit-exact against the oracle; the step
API with host-written levels (current_level / previous_level mirrors
scattered to and gathered from the slabs) bit-exact against one domain;
max_abs reduced over the slabs; one verbose line per health check."""
import re

import numpy as np
import pytest

from helpers import D, N, X, gpu_solver, oracle_solver, rel_l2, same, small_config
from paper_2201_05278_b200 import DampingField, SlabSolver, Solver, make_material_model
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu


def _slab(w, devices):
    return Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
                  devices=devices)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_forward_matches_the_oracle(devices):
    h = 20.0
    cfg = small_config(ndim=3, order=8, shape=(41, 27, 25), bc=[[N, D], [D, X], [D, N]], n_rec=9,
                       src=[(h * 20.5, h * 13.5, h * 12.5)], steps=60)
    # receiver lines across the slab faces (extended planes 25 | 26 and 33 | 34)
    cfg.receivers = ([(h * 20.5, h * (2.5 + 2 * k), h * 12.5) for k in range(10)]
                     + [(h * 28.5, h * (3.5 + 2 * k), h * 11.5) for k in range(10)])
    w = build_workload(cfg, np.float32)
    s = _slab(w, devices)
    assert isinstance(s, SlabSolver) and s.devices() == devices
    s.set_sources(w.sources, w.wavelet)
    s.set_receivers(w.receivers)
    res = s.forward()
    from paper_2201_05278_b200.dist import split_products
    assert sum(len(split_products(r, 61)[0]) for r in s._ranks) > 0  # straddling taps exist
    s.close()
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    assert np.abs(ref["final"]).max() > 0
    assert same(res.snapshots[-1], ref["final"])
    # receivers whose taps straddle a slab face are merged from per-tap products
    assert same(np.asarray(res.seismogram.data), ref["seismogram"])


def test_step_api_and_max_abs_match_one_domain():
    cfg = small_config(ndim=3, order=4, shape=(33, 21, 19), steps=30, bc=[[D, N], [N, D], [X, D]])
    w = build_workload(cfg, np.float32)
    rng = np.random.default_rng(3)
    a = rng.standard_normal(w.velocity.shape).astype(np.float32)
    b = rng.standard_normal(w.velocity.shape).astype(np.float32)
    one = gpu_solver(w)
    two = _slab(w, [0, 0])
    for s in (one, two):
        s.previous_level()[...] = a
        s.current_level()[...] = b
        s.refresh_boundary()
    for _ in range(7):
        one.step()
        two.step()
        assert same(two.current_level(), one.current_level())
        assert same(two.previous_level(), one.previous_level())
    assert two.step_index() == one.step_index() == 7
    assert two.max_abs() == one.max_abs()
    one.close()
    two.close()


def test_verbose_line_once_per_check(capsys):
    w = build_workload(small_config(ndim=3, order=4, shape=(31, 17, 15), steps=150), np.float32)
    s = _slab(w, [0, 0])
    s.set_sources(w.sources, w.wavelet)
    s.set_verbose(True)
    s.forward()
    s.close()
    lines = [l for l in capsys.readouterr().err.splitlines() if re.match(r"^step \d+/150  ", l)]
    assert [l.split()[1] for l in lines] == ["100/150", "150/150"]
