"""The reference's hot-path tests (proj/tests/test_kernel.cpp) restated in
Python and run against two backends: the CPU oracle (`-m "not gpu"`) and the
GPU Solver through the C-ABI (`-m gpu`).  Every Solver here is double
precision, as in the reference tests (test_kernel.cpp:37)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2201_05278_b200 import (BoundaryCondition, BoundarySpec, InstabilityError, Solver, TimeAxis,
                                   build_grid, build_injection_map, damping_field, extend_with_damping,
                                   make_material_model, make_point_set, make_stencil, ricker_samples,
                                   stable_dt)
from paper_2201_05278_b200.grid import Precision

BC = BoundaryCondition


class OracleAPI:
    """The oracle behind the reference Solver's method names."""

    def __init__(self, grid, materials, damping, spec, axis, coeffs):
        self._s = O.OracleSolver(grid.ndim, grid.space_order, np.float64, grid.extended_shape, grid.spacing,
                                 axis.dt, axis.n_steps, spec.face, materials.velocity, damping.eta,
                                 density=materials.density)
        self._axis = axis
        self._grid = grid
        self._n_rec = 0

    def current_level(self):
        return self._s.current()

    def previous_level(self):
        return self._s.previous()

    def refresh_boundary(self):
        self._s.refresh_boundary()

    def step(self):
        bad = self._s.step()
        if bad:
            raise InstabilityError(*bad)

    def max_abs(self):
        return self._s.max_abs()

    def set_sources(self, m, w):
        self._s.set_sources(m, w)

    def set_receivers(self, m, coords=None):
        self._s.set_receivers(m)
        self._n_rec = m.n_points

    def set_backend(self, *a):
        pass

    def grid(self):
        return self._grid

    def forward(self):
        r = self._s.forward()
        if "unstable" in r:
            raise InstabilityError(*r["unstable"])

        class R:
            pass
        out = R()
        out.seismogram = R()
        out.seismogram.data = r["seismogram"]
        out.seismogram.n_receivers = self._n_rec
        out.snapshots = [r["final"]]
        out.snapshot_steps = [self._axis.n_steps]
        return out


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def backend(request):
    return request.param


def make_solver(backend, extent_z=8.0, extent_x=8.0, h=1.0, c=1.0, order=2, dt=0.1, steps=1,
                damping_length=0.0, alpha=0.0, power=3.0, bc=BC.None_, stride=0, rho=None):
    """test_kernel.cpp:37-66 make_solver."""
    grid = build_grid([0, extent_z, 0, extent_x], [h, h], order, Precision.Double)
    grid = extend_with_damping(grid, [damping_length] * 4)
    vel = np.full(grid.padded_shape()[:2], c, np.float64)
    mats = make_material_model(vel, None if rho is None else np.full_like(vel, rho))
    damp = damping_field(grid, alpha, power, np.float64)
    axis = TimeAxis(tf=dt * steps, dt=dt, n_steps=steps, saving_stride=stride,
                    stable_bound=stable_dt(c, [h, h], order, 2))
    cls = Solver if backend == "gpu" else OracleAPI
    return cls(grid, mats, damp, BoundarySpec.uniform(bc), axis, make_stencil(order))


def test_zero_field_zero_source_stays_zero(backend):  # test_kernel.cpp:70-74
    s = make_solver(backend)
    s.step()
    assert np.all(s.current_level() == 0.0)


def test_hand_computed_impulse_response(backend):  # :76-100
    s = make_solver(backend)
    cz = cx = 1 + 4
    s.current_level()[cz, cx] = 1.0
    s.refresh_boundary()
    s.step()
    c2dt2 = 0.01
    nxt = s.current_level()
    assert abs(nxt[cz, cx] - (2.0 + c2dt2 * -4.0)) <= 1e-15
    for dz, dx in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        assert abs(nxt[cz + dz, cx + dx] - c2dt2) <= 1e-15
    assert nxt[cz + 1, cx + 1] == 0.0 and nxt[cz - 1, cx - 1] == 0.0 and nxt[cz + 2, cx] == 0.0
    assert s.previous_level()[cz, cx] == 1.0


def test_dirichlet_forces_face_and_mirrors_ghosts(backend):  # :125-137
    s = make_solver(backend, bc=BC.NullDirichlet)
    cur = s.current_level()
    iz, ix = np.meshgrid(np.arange(cur.shape[0]), np.arange(cur.shape[1]), indexing="ij")
    cur[...] = 1.0 + iz * 0.1 + ix * 0.01
    s.refresh_boundary()
    cur = s.current_level()
    assert cur[1, 5] == 0.0 and cur[0, 5] == -cur[2, 5]
    assert cur[9, 5] == 0.0 and cur[10, 5] == -cur[8, 5]


def test_neumann_mirrors_and_none_zero_fills(backend):  # :139-157
    s = make_solver(backend, bc=BC.NullNeumann)
    cn = s.current_level()
    iz, ix = np.meshgrid(np.arange(cn.shape[0]), np.arange(cn.shape[1]), indexing="ij")
    cn[...] = iz + 100.0 * ix
    s.refresh_boundary()
    cn = s.current_level()
    assert cn[0, 5] == cn[2, 5] and cn[10, 5] == cn[8, 5] and cn[5, 0] == cn[5, 2]
    s2 = make_solver(backend, bc=BC.None_)
    cz = s2.current_level()
    cz[...] = 3.0
    s2.refresh_boundary()
    cz = s2.current_level()
    assert cz[0, 5] == 0.0 and cz[10, 5] == 0.0 and cz[1, 5] == 3.0


def test_dirichlet_boundary_trace_stays_zero(backend):  # :159-176
    s = make_solver(backend, extent_z=30, extent_x=30, dt=0.2, steps=50, bc=BC.NullDirichlet)
    s.current_level()[8, 9] = 1.0
    s.refresh_boundary()
    for _ in range(50):
        s.step()
        f = s.current_level()
        assert np.all(f[1, 1:30] == 0) and np.all(f[31, 1:30] == 0)
        assert np.all(f[1:30, 1] == 0) and np.all(f[1:30, 31] == 0)


def test_neumann_preserves_mirror_symmetry(backend):  # :178-197
    s = make_solver(backend, extent_z=24, extent_x=24, dt=0.2, steps=40, bc=BC.NullNeumann)
    cur = s.current_level()
    iz, ix = np.meshgrid(np.arange(cur.shape[0]), np.arange(cur.shape[1]), indexing="ij")
    cur[...] = np.exp(-((iz - 13.0) ** 2 + (ix - 13.0) ** 2) / 8.0)
    s.refresh_boundary()
    for _ in range(40):
        s.step()
    f = s.current_level()
    inner = f[1:-1, 1:-1]
    assert np.array_equal(inner, inner[::-1, :]) and np.array_equal(inner, inner[:, ::-1])


def test_dirichlet_reflects_with_inverted_sign(backend):  # :199-245
    grid = build_grid([0, 4, 0, 400], [1, 1], 2, Precision.Double)
    grid = extend_with_damping(grid, [0, 0, 0, 0])
    vel = np.ones(grid.padded_shape()[:2])
    axis = TimeAxis(tf=170.0, dt=0.5, n_steps=340, stable_bound=stable_dt(1.0, [1, 1], 2, 2))
    spec = BoundarySpec([[BC.NullNeumann] * 2, [BC.NullDirichlet] * 2, [BC.NullDirichlet] * 2])
    cls = Solver if backend == "gpu" else OracleAPI
    s = cls(grid, make_material_model(vel), damping_field(grid, 0.0, 0.0, np.float64), spec, axis,
            make_stencil(2))
    x = np.arange(grid.padded_shape()[1]) - 1.0
    s.current_level()[...] = np.exp(-(x - 320.0) ** 2 / 200.0)[None, :]
    s.previous_level()[...] = np.exp(-(x - 320.0 + 0.5) ** 2 / 200.0)[None, :]
    s.refresh_boundary()
    probe_min, min_step = 1.0, 0
    for n in range(340):
        s.step()
        v = s.current_level()[3, 321]
        if v < probe_min:
            probe_min, min_step = v, n + 1
    assert probe_min < -0.7
    assert min_step > 250


def test_seismogram_row_count_and_quiescent_start(backend):  # :342-356
    s = make_solver(backend, extent_z=40, extent_x=40, dt=0.2, steps=25, bc=BC.NullDirichlet)
    g = s.grid()
    s.set_sources(build_injection_map(make_point_set([(20, 20, 0)], 4), g), ricker_samples(26, 0.2, 0.5))
    s.set_receivers(build_injection_map(make_point_set([(20, 26, 0)], 4), g))
    r = s.forward()
    assert r.seismogram.n_receivers == 1
    assert len(r.seismogram.data) == 26
    assert r.seismogram.data[0] == 0.0


def _linear_run(backend, scale):
    s = make_solver(backend, extent_z=60, extent_x=60, dt=0.2, steps=120, bc=BC.NullDirichlet)
    g = s.grid()
    w = ricker_samples(121, 0.2, 0.25) * scale
    s.set_sources(build_injection_map(make_point_set([(30, 30, 0)], 4), g), w)
    s.set_receivers(build_injection_map(make_point_set([(30, 45.5, 0)], 4), g))
    return np.asarray(s.forward().seismogram.data)


def test_linearity_in_the_source(backend):  # :358-380
    base = _linear_run(backend, 1.0)
    doubled = _linear_run(backend, 2.0)
    peak = np.abs(base).max()
    assert peak > 0
    assert np.all(np.abs(doubled - 2.0 * base) <= peak * 2.0 * 1e-10)


def test_time_reversal_recovers_initial_state(backend):  # :382-411
    kw = dict(extent_z=30, extent_x=30, dt=0.2, steps=1, bc=BC.NullDirichlet)
    fw = make_solver(backend, **kw)
    cur = fw.current_level()
    iz, ix = np.meshgrid(np.arange(cur.shape[0]), np.arange(cur.shape[1]), indexing="ij")
    cur[...] = np.exp(-((iz - 15.0) ** 2 + (ix - 16.0) ** 2) / 12.0)
    fw.refresh_boundary()
    p0 = fw.current_level().copy()
    for _ in range(60):
        fw.step()
    pk, pk1 = fw.current_level().copy(), fw.previous_level().copy()
    bw = make_solver(backend, **kw)
    bw.current_level()[...] = pk1
    bw.previous_level()[...] = pk
    bw.refresh_boundary()
    for _ in range(59):
        bw.step()
    assert np.abs(bw.current_level() - p0).max() < 1e-11


def _stability_run(backend, dt, max_steps):
    s = make_solver(backend, extent_z=400, extent_x=400, h=10.0, c=1500.0, dt=dt, steps=max_steps,
                    bc=BC.NullDirichlet)
    s.set_sources(build_injection_map(make_point_set([(200, 200, 0)], 4), s.grid()),
                  ricker_samples(max_steps + 1, dt, 15.0))
    driven = glob = 0.0
    for n in range(max_steps):
        s.step()
        m = s.max_abs()
        if n < 500:
            driven = max(driven, m)
        glob = max(glob, m)
    return driven, glob


def test_stability_bounded_then_blows_up(backend):  # :413-456
    dts = stable_dt(1500.0, [10.0, 10.0], 2, 2)
    driven, glob = _stability_run(backend, dts, 2000)
    assert driven > 0 and glob <= 10.0 * driven
    with pytest.raises(InstabilityError) as ei:
        _stability_run(backend, 1.5 * dts, 2000)
    assert ei.value.step() < 2000 and ei.value.step() % 100 == 0


def test_damping_energy_decreases_with_alpha(backend):  # :458-479
    def energy(alpha):
        s = make_solver(backend, extent_z=200, extent_x=200, h=5.0, c=1500.0, order=2, dt=2e-3, steps=250,
                        damping_length=100.0, alpha=alpha, power=3.0, bc=BC.NullDirichlet)
        s.set_sources(build_injection_map(make_point_set([(100, 100, 0)], 4), s.grid()),
                      ricker_samples(251, 2e-3, 25.0))
        s.forward()
        return float(np.sum(np.asarray(s.current_level(), np.float64) ** 2))
    e0, e1, e2 = energy(0.0), energy(1e-5), energy(1e-4)
    assert e0 > e1 > e2


def test_backends_identical(backend):  # :481-504 (set_backend is a no-op on the GPU)
    def run():
        s = make_solver(backend, extent_z=100, extent_x=100, h=2.0, c=1500.0, order=8, dt=5e-4, steps=80,
                        bc=BC.NullDirichlet)
        s.set_backend(1, 4)
        s.set_sources(build_injection_map(make_point_set([(50, 50, 0)], 4), s.grid()),
                      ricker_samples(81, 5e-4, 20.0))
        s.set_receivers(build_injection_map(make_point_set([(50, 80, 0)], 4), s.grid()))
        return np.asarray(s.forward().seismogram.data)
    a, b = run(), run()
    assert np.abs(a).max() > 0 and np.array_equal(a, b)


@pytest.mark.gpu
def test_tf_smaller_than_dt_runs_one_step():  # :305-311
    s = make_solver("gpu", extent_z=20, extent_x=20, steps=1)
    r = s.forward()
    assert len(r.snapshots) == 1 and r.snapshot_steps[0] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("stride", [0, 1, 3, 7])
def test_snapshot_stride_bookkeeping(stride):  # :313-340
    s = make_solver("gpu", extent_z=20, extent_x=20, dt=0.2, steps=20, stride=stride)
    r = s.forward()
    expect = 1 if stride == 0 else 20 // stride + 1
    assert len(r.snapshots) == expect
    for snap in r.snapshots:
        assert snap.shape == (s.grid().extended_shape[0], s.grid().extended_shape[1])
    if stride:
        assert r.snapshot_steps == list(range(0, 21, stride))


@pytest.mark.gpu
def test_snapshot_memory_guard():  # :506-520
    s = make_solver("gpu", extent_z=100, extent_x=100, dt=0.2, steps=50, stride=1)
    s.set_snapshot_cap(1024)
    with pytest.raises(ValueError):
        s.forward()


def test_constant_density_equals_variable_density_with_constant_rho(backend):  # :102-123
    runs = []
    for rho in (None, 2.7):
        s = make_solver(backend, extent_z=40, extent_x=40, dt=0.2, steps=30, bc=BC.NullDirichlet, rho=rho)
        cur = s.current_level()
        iz, ix = np.meshgrid(np.arange(cur.shape[0]), np.arange(cur.shape[1]), indexing="ij")
        cur[...] = np.exp(-((iz - 20.0) ** 2 + (ix - 20.0) ** 2) / 18.0)
        s.refresh_boundary()
        for _ in range(30):
            s.step()
        runs.append(np.array(s.current_level()))
    assert np.array_equal(runs[0], runs[1])  # grad(rho) is exactly zero
