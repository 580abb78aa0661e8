"""GPU (libfdwave_cuda.so) vs the CPU oracle on identical inputs.

EXACT arithmetic mode is IEEE-identical to the reference (no FMA, same
association), so seismograms, final levels and the full padded levels
(ghosts included) must be EQUAL.  FMA mode is held to rel-L2 1e-5 here.
"""
import numpy as np
import pytest

from helpers import D, N, X, gpu_solver, oracle_solver, rel_l2, run_both, same, small_config
from paper_2201_05278_b200 import InstabilityError
from paper_2201_05278_b200._lib import (FDW_KERNEL_FUSED2D, FDW_KERNEL_SIMPLE, FDW_KERNEL_TMA, FDW_KERNEL_ZMARCH,
                                        FDW_MATH_FMA)
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu

BCS = [
    [[N, D], [D, D], [D, D]],
    [[D, D], [N, N], [X, D]],
    [[X, X], [X, N], [N, X]],
]


@pytest.mark.parametrize("order", [2, 4, 8, 12, 20])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("bci", range(3))
@pytest.mark.parametrize("variant", [FDW_KERNEL_SIMPLE, FDW_KERNEL_FUSED2D])
def test_2d_exact(order, dtype, bci, variant):
    cfg = small_config(ndim=2, order=order, shape=(37, 53), damping_cells=6, bc=BCS[bci], tf=0.25)
    w, g, res, o, ref = run_both(cfg, dtype, variant=variant)
    assert w.axis.n_steps > 20
    assert same(res.seismogram.data, ref["seismogram"])
    assert same(res.snapshots[-1], ref["final"])
    assert same(g.current_level(), o.current())
    assert same(g.previous_level(), o.previous())
    assert np.abs(ref["final"]).max() > 0


@pytest.mark.parametrize("order", [2, 4, 6, 8])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("variant", [FDW_KERNEL_SIMPLE, FDW_KERNEL_ZMARCH, FDW_KERNEL_TMA])
@pytest.mark.parametrize("bci", range(3))
def test_3d_exact(order, dtype, variant, bci):
    cfg = small_config(ndim=3, order=order, shape=(17, 27, 21), damping_cells=4, bc=BCS[bci], tf=0.12)
    w, g, res, o, ref = run_both(cfg, dtype, variant=variant)
    assert w.axis.n_steps > 20
    assert same(res.seismogram.data, ref["seismogram"])
    assert same(res.snapshots[-1], ref["final"])
    assert same(g.current_level(), o.current())
    assert same(g.previous_level(), o.previous())


@pytest.mark.parametrize("shape", [(13, 33, 65), (29, 17, 69), (12, 49, 7), (40, 18, 131)])
@pytest.mark.parametrize("zseg", [1, 3, 7])
@pytest.mark.parametrize("variant", [FDW_KERNEL_ZMARCH, FDW_KERNEL_TMA])
def test_3d_zmarch_ragged_tiles(shape, zseg, variant):
    """Partial Y vectors / X tiles / Z segments all cover the grid exactly once."""
    cfg = small_config(ndim=3, order=8, shape=shape, damping_cells=3, tf=0.06)
    w, g, res, o, ref = run_both(cfg, np.float32, variant=variant, z_segments=zseg)
    assert same(res.seismogram.data, ref["seismogram"])
    assert same(res.snapshots[-1], ref["final"])
    assert same(g.current_level(), o.current())


@pytest.mark.parametrize("ndim", [2, 3])
def test_fma_mode_within_tolerance(ndim):
    shape = (37, 53) if ndim == 2 else (17, 27, 21)
    cfg = small_config(ndim=ndim, order=8, shape=shape, tf=0.25 if ndim == 2 else 0.12)
    w, g, res, o, ref = run_both(cfg, np.float32, math=FDW_MATH_FMA)
    assert rel_l2(res.seismogram.data, ref["seismogram"]) < 1e-5
    assert rel_l2(res.snapshots[-1], ref["final"]) < 1e-5


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("bci", range(3))
def test_step_api_random_levels(ndim, bci):
    """(default variants: FUSED2D in 2D, TMA in 3D -- both take the stored-ghost
    path for the first step after an upload)"""
    """Host-mirror semantics: write both levels, refresh, step -- levels equal
    the oracle's (ghosts included) after every step."""
    shape = (21, 25) if ndim == 2 else (14, 17, 19)
    cfg = small_config(ndim=ndim, order=4, shape=shape, bc=BCS[bci], tf=0.05)
    w = build_workload(cfg, np.float64)
    g = gpu_solver(w)
    o = oracle_solver(w)
    rng = np.random.default_rng(7)
    a = rng.standard_normal(o.current().shape)
    b = rng.standard_normal(o.current().shape)
    g.current_level()[...] = a
    g.previous_level()[...] = b
    o.current()[...] = a
    o.previous()[...] = b
    g.refresh_boundary()
    o.refresh_boundary()
    assert same(g.current_level(), o.current())
    for _ in range(5):
        g.step()
        o.step()
        assert same(g.current_level(), o.current())
        assert same(g.previous_level(), o.previous())
        assert g.max_abs() == o.max_abs()
    assert g.step_index() == o.step_index() == 5


@pytest.mark.parametrize("ndim", [2, 3])
def test_instability_is_reported_at_the_same_step(ndim):
    shape = (41, 41) if ndim == 2 else (15, 15, 15)
    cfg = small_config(ndim=ndim, order=2, shape=shape, damping_cells=0, tf=0.5,
                       bc=[[D, D], [D, D], [D, D]])
    w = build_workload(cfg, np.float32)
    w.axis.dt *= 1.5
    w.axis.n_steps = 1000
    w.wavelet = np.resize(w.wavelet, 1001)
    g = gpu_solver(w)
    g.set_sources(w.sources, w.wavelet)
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    bad = None
    for _ in range(1000):
        bad = o.step()
        if bad:
            break
    assert bad is not None
    with pytest.raises(InstabilityError) as ei:
        g.advance_raw(1000)
    assert ei.value.step() == bad[0]
    assert np.isnan(ei.value.max_abs()) == np.isnan(bad[1])
    assert g.step_index() == bad[0]


def test_two_solvers_interleaved():
    """Contexts are independent (coefficients travel as launch parameters)."""
    c1 = small_config(ndim=3, order=8, shape=(15, 19, 17), tf=0.06)
    c2 = small_config(ndim=2, order=4, shape=(30, 40), tf=0.1)
    w1, w2 = build_workload(c1, np.float32), build_workload(c2, np.float64)
    g1, g2 = gpu_solver(w1), gpu_solver(w2)
    for g, w in ((g1, w1), (g2, w2)):
        g.set_sources(w.sources, w.wavelet)
        g.set_receivers(w.receivers)
    r1 = g1.forward()
    r2 = g2.forward()
    for w, r in ((w1, r1), (w2, r2)):
        o = oracle_solver(w)
        o.set_sources(w.sources, w.wavelet)
        o.set_receivers(w.receivers)
        ref = o.forward()
        assert same(r.seismogram.data, ref["seismogram"])


def test_verbose_progress_line(capsys):
    """Solver.set_verbose(True): the reference's line at every health check
    (kernel.hpp:456-466), "step s/N  t s  max|p| = m", with max|p| the
    oracle's max_abs at that step."""
    import re
    w = build_workload(small_config(ndim=3, order=4, shape=(19, 23, 21), steps=230), np.float32)
    g = gpu_solver(w)
    g.set_sources(w.sources, w.wavelet)
    g.set_verbose(True)
    g.forward()
    err = capsys.readouterr().err
    pat = re.compile(r"^step (\d+)/(\d+)  \d+\.\d{3}s  max\|p\| = (\S+)$")
    lines = [m.groups() for m in (pat.match(l) for l in err.splitlines()) if m]
    assert [int(a) for a, _, _ in lines] == [100, 200, 230] and all(b == "230" for _, b, _ in lines)
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.refresh_boundary()
    want = []
    for k in range(1, 231):
        o.step()
        if k % 100 == 0 or k == 230:
            want.append("%.6e" % o.max_abs())
    assert [m for _, _, m in lines] == want


@pytest.mark.parametrize("n_distinct", [7, 255, 256, 5000])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_damping_table_and_fallback(n_distinct, dtype):
    """The TMA sweep (fp32 and fp64) streams a 1-byte damping index with a
    (1 - eta dt, 1/(1 + eta dt)) table when eta has <= 255 distinct non-zero
    values, and T(eta) otherwise: both bit-exact against the oracle, on an eta
    field with arbitrary values everywhere (not just an absorbing shell)."""
    cfg = small_config(ndim=3, order=8, shape=(23, 27, 70), steps=40, n_rec=8)
    w = build_workload(cfg, dtype)
    rng = np.random.default_rng(n_distinct)
    values = rng.uniform(1.0, 60.0, n_distinct).astype(dtype)
    eta = values[rng.integers(0, n_distinct, w.eta.shape)]
    eta[rng.random(w.eta.shape) < 0.5] = 0.0  # undamped points interleaved
    w.eta = np.ascontiguousarray(eta)
    g = gpu_solver(w)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    assert np.abs(ref["final"]).max() > 0
    assert same(res.snapshots[-1], ref["final"])
    assert same(np.asarray(res.seismogram.data), ref["seismogram"])
