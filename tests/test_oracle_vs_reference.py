"""The C restatement (oracle/liboracle.so) against the reference compiled in
place (oracle/_ref/libfdwave_ref.so): bit-identical on every piece of the
path.  Skipped only when the reference library was never built."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from helpers import D, N, X, same

REF = O.rlib()
pytestmark = pytest.mark.skipif(REF is None, reason="oracle/_ref not built (reference tree absent)")


@pytest.mark.parametrize("order", range(2, 22, 2))
def test_coefficients_and_cfl(order):
    v_ref = np.zeros(order // 2 + 1)
    REF.ref_second_derivative(order, v_ref.ctypes.data_as(C.c_void_p))
    v_or = np.zeros(11)
    O.olib().fdwo_second_derivative_coefficients(order, v_or.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(v_ref, v_or[: order // 2 + 1])
    for ndim, sp in ((2, [10.0, 7.5]), (3, [20.0, 20.0, 12.5])):
        s = np.asarray(sp)
        a = REF.ref_stable_dt(4700.0, s.ctypes.data_as(C.c_void_p), len(sp), order, ndim)
        b = O.olib().fdwo_stable_dt(4700.0, s.ctypes.data_as(C.POINTER(C.c_double)), len(sp), order, ndim)
        assert a == b


def test_special_functions_and_ricker():
    L = O.olib()
    for x in np.linspace(-40, 140, 997):
        assert REF.ref_bessel_i0(x) == L.fdwo_bessel_i0(x)
    for x in list(np.linspace(-7.3, 7.3, 1001)) + [0.0, 1.0, -3.0, 1e-6, 2.5e-5]:
        assert REF.ref_sinc(x) == L.fdwo_sinc(x)
    a = np.zeros(3001)
    b = np.zeros(3001)
    REF.ref_ricker(3001, 1.509518e-3, 10.0, a.ctypes.data_as(C.c_void_p))
    L.fdwo_ricker_samples(3001, 1.509518e-3, 10.0, b.ctypes.data_as(C.c_void_p))
    assert np.array_equal(a, b)


def _pair(ndim, order, dtype, ext, bc, seed, eta_scale=0.0):
    rng = np.random.default_rng(seed)
    pad = tuple(e + order for e in ext)
    vel = (1500 + 3000 * rng.random(pad)).astype(dtype)
    eta = (eta_scale * rng.random(pad)).astype(dtype)
    sp = [10.0, 12.0, 9.0][:ndim]
    dt = 0.3 * 9.0 / 4500.0
    args = (ndim, order, dtype, ext, sp, dt, 250, bc, vel, eta)
    return O.RefSolver(*args), O.OracleSolver(*args)


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("order", [2, 4, 8, 14])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("bc", [[[N, D], [D, D], [D, D]], [[X, N], [D, X], [N, N]]])
def test_step_api_random_state(ndim, order, dtype, bc):
    ext = (12, 14) if ndim == 2 else (11, 12, 13)
    ext = tuple(e + order for e in ext)
    r, o = _pair(ndim, order, dtype, ext, bc, seed=order + ndim, eta_scale=30.0)
    rng = np.random.default_rng(1)
    a = rng.standard_normal(r.shape).astype(dtype)
    b = rng.standard_normal(r.shape).astype(dtype)
    for s in (r, o):
        s.current()[...] = a
        s.previous()[...] = b
        s.refresh_boundary()
    for _ in range(6):
        assert r.step() == o.step()
        assert same(r.current(), o.current())
        assert same(r.previous(), o.previous())
        assert r.max_abs() == o.max_abs()


def test_first_non_finite_is_reported_like_the_reference():
    r, o = _pair(2, 4, np.float32, (20, 20), [[D, D], [D, D], [D, D]], seed=3)
    for s in (r, o):
        s.current()[5, 7] = np.inf
        s.current()[3, 9] = np.nan
    assert np.isnan(r.max_abs()) and np.isnan(o.max_abs())


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("order", [2, 4, 8])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_variable_density_branch(ndim, order, dtype):
    """VariableDensity = true: density_log_gradient + the extra sweep terms
    (kernel.hpp:104-136, :365-373, :407-417), bit-identical."""
    ext = (14, 16) if ndim == 2 else (12, 13, 14)
    ext = tuple(e + order for e in ext)
    rng = np.random.default_rng(11 + order)
    pad = tuple(e + order for e in ext)
    vel = (1500 + 3000 * rng.random(pad)).astype(dtype)
    eta = (20.0 * rng.random(pad)).astype(dtype)
    rho = (1.0 + 2.0 * rng.random(pad)).astype(dtype)
    sp = [10.0, 12.0, 9.0][:ndim]
    args = (ndim, order, dtype, ext, sp, 0.3 * 9.0 / 4500.0, 250, [[N, D], [X, D], [D, N]], vel, eta)
    r, o = O.RefSolver(*args, density=rho), O.OracleSolver(*args, density=rho)
    g_ref = np.zeros((3,) + pad, dtype)
    REF.ref_density_log_gradient(ndim, order, np.dtype(dtype).itemsize,
                                 np.array(list(ext) + [1] * (3 - ndim), np.uint64).ctypes.data_as(C.c_void_p),
                                 np.array(sp + [1.0] * (3 - ndim)).ctypes.data_as(C.c_void_p),
                                 rho.ctypes.data_as(C.c_void_p), g_ref.ctypes.data_as(C.c_void_p))
    g_or = np.zeros((3,) + pad, dtype)
    grid = O.fdwo_grid()
    grid.ndim, grid.halo, grid.space_order = ndim, order // 2, order
    for a in range(3):
        grid.spacing[a] = sp[a] if a < ndim else 1.0
        grid.extended[a] = ext[a] if a < ndim else 1
        grid.padded[a] = pad[a] if a < ndim else 1
    O.olib().fdwo_density_log_gradient(C.byref(grid), np.dtype(dtype).itemsize, rho.ctypes.data_as(C.c_void_p),
                                       g_or.ctypes.data_as(C.c_void_p))
    assert same(g_ref[:ndim], g_or[:ndim])
    a = rng.standard_normal(r.shape).astype(dtype)
    for s_ in (r, o):
        s_.current()[...] = a
        s_.refresh_boundary()
    for _ in range(5):
        assert r.step() == o.step()
        assert same(r.current(), o.current())


@pytest.mark.parametrize("ndim,order", [(2, 4), (3, 8)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_volume_sources(ndim, order, dtype):
    """Dense modulated sources (kernel.hpp:439-452) after the point sources,
    two of them in insertion order, plus the amplitude-length check (:199-203)."""
    ext = (14, 16) if ndim == 2 else (12, 13, 14)
    pad = tuple(e + order for e in ext)
    rng = np.random.default_rng(5 + order)
    vel = (1500 + 3000 * rng.random(pad)).astype(dtype)
    eta = (20.0 * rng.random(pad)).astype(dtype)
    sp = [10.0, 12.0, 9.0][:ndim]
    steps = 12
    args = (ndim, order, dtype, ext, sp, 0.3 * 9.0 / 4500.0, steps, [[N, D], [X, D], [D, N]], vel, eta)
    r, o = O.RefSolver(*args), O.OracleSolver(*args)
    f1 = rng.standard_normal(pad).astype(dtype)
    f2 = rng.standard_normal(pad).astype(dtype)
    a1 = np.sin(np.arange(steps + 3) * 0.7)
    a2 = np.cos(np.arange(steps) * 0.3) * 1e3
    for s_ in (r, o):
        s_.add_volume_source(f1, a1)
        s_.add_volume_source(f2, a2)
        with pytest.raises(ValueError):
            s_.add_volume_source(f2, a2[:-1])
    for _ in range(steps):
        r.step()
        o.step()
        assert same(r.current(), o.current()) and same(r.previous(), o.previous())
    assert np.abs(o.current()).max() > 0
