"""Variable density on the CUDA path (MaterialModel::density, kernel.hpp:104-136
density_log_gradient, sweep terms :365-373 (2D) / :407-417 (3D)) against the
oracle's VariableDensity = true branch, bit-exact; plus the reference's own
test_kernel.cpp linked against the drop-in header (oracle/_ref/test_kernel_cuda)."""
import os
import subprocess

import numpy as np
import pytest

from helpers import D, N, X, oracle_solver, same, small_config
import oracle as O
from paper_2201_05278_b200 import DampingField, Solver, make_material_model
from paper_2201_05278_b200._lib import FDW_KERNEL_SIMPLE, FDW_KERNEL_TMA, FDW_KERNEL_ZMARCH
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def density_field(shape, dtype, seed):
    """Smooth-ish positive density (g/cm^3) with a sharp layer, padded grid."""
    rng = np.random.default_rng(seed)
    rho = 1.5 + 0.8 * rng.random(shape)
    rho[: shape[0] // 2] += 0.7  # a contrast the gradient stencil must see
    return rho.astype(dtype)


def run_vd(cfg, dtype, seed=3, **kw):
    w = build_workload(cfg, dtype)
    rho = density_field(w.velocity.shape, dtype, seed)
    g = Solver(w.grid, make_material_model(w.velocity, rho), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
               **kw)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    o = O.OracleSolver(w.grid.ndim, w.grid.space_order, w.velocity.dtype, w.grid.extended_shape, w.grid.spacing,
                       w.axis.dt, w.axis.n_steps, w.spec.face, w.velocity, w.eta, density=rho)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    return w, g, res, ref


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("order", [2, 4, 8, 16, 20])
def test_vd_2d_forward(order, dtype):
    cfg = small_config(ndim=2, order=order, shape=(41, 53), bc=[[N, D], [D, N], [D, D]])
    w, g, res, ref = run_vd(cfg, dtype)
    assert np.abs(ref["final"]).max() > 0
    assert same(res.seismogram.data, ref["seismogram"])
    assert same(res.snapshots[-1], ref["final"])


@pytest.mark.parametrize("variant", [0, FDW_KERNEL_SIMPLE, FDW_KERNEL_ZMARCH, FDW_KERNEL_TMA])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("order", [2, 4, 8, 12])
def test_vd_3d_forward(order, dtype, variant):
    cfg = small_config(ndim=3, order=order, shape=(21, 27, 25), bc=[[N, D], [D, X], [D, N]])
    w, g, res, ref = run_vd(cfg, dtype, variant=variant)
    # density terms: the TMA sweep keeps its kernel (3 gradient tiles more);
    # the other 3D variants fall back to the element-wise sweep
    tma_built = order // 2 in (1, 2, 4)
    want = FDW_KERNEL_TMA if variant in (0, FDW_KERNEL_TMA) and tma_built else FDW_KERNEL_SIMPLE
    assert g.layout()["variant"] == want
    assert np.abs(ref["final"]).max() > 0
    assert same(res.seismogram.data, ref["seismogram"])
    assert same(res.snapshots[-1], ref["final"])


def test_vd_constant_rho_equals_constant_density():
    """kernel.hpp test Step.ConstantDensityEqualsVariableDensityWithConstantRho
    on the GPU: grad(rho)/rho == 0 so the density branch changes nothing."""
    cfg = small_config(ndim=3, order=8, shape=(19, 23, 21))
    w = build_workload(cfg, np.float64)
    outs = []
    for rho in (None, np.full(w.velocity.shape, 2.2, np.float64)):
        g = Solver(w.grid, make_material_model(w.velocity, rho), DampingField(eta=w.eta), w.spec, w.axis,
                   w.coeffs)
        g.set_sources(w.sources, w.wavelet)
        g.set_receivers(w.receivers)
        outs.append(g.forward())
    assert same(outs[0].seismogram.data, outs[1].seismogram.data)
    assert same(outs[0].snapshots[-1], outs[1].snapshots[-1])


@pytest.mark.parametrize("ndim", [2, 3])
def test_vd_raw_levels_step_by_step(ndim):
    """Initial conditions written through the level mirrors, then single steps
    (Solver::step, kernel.hpp:226-233) with the density terms."""
    shape = (17, 19) if ndim == 2 else (15, 17, 16)
    cfg = small_config(ndim=ndim, order=6, shape=shape, bc=[[D, N], [N, D], [X, D]])
    w = build_workload(cfg, np.float32)
    rho = density_field(w.velocity.shape, np.float32, 9)
    g = Solver(w.grid, make_material_model(w.velocity, rho), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
    o = O.OracleSolver(ndim, 6, np.float32, w.grid.extended_shape, w.grid.spacing, w.axis.dt, w.axis.n_steps,
                       w.spec.face, w.velocity, w.eta, density=rho)
    a = np.random.default_rng(5).standard_normal(o.shape).astype(np.float32)
    g.current_level()[...] = a
    g.refresh_boundary()
    o.current()[...] = a
    o.refresh_boundary()
    for _ in range(6):
        g.step()
        o.step()
        assert same(g.current_level(), o.current())
        assert same(g.previous_level(), o.previous())


def test_vd_rejects_shape_mismatch():
    cfg = small_config(ndim=2, order=4, shape=(17, 19))
    w = build_workload(cfg, np.float32)
    with pytest.raises(ValueError):
        Solver(w.grid, make_material_model(w.velocity, np.ones(7, np.float32)), DampingField(eta=w.eta), w.spec,
               w.axis, w.coeffs)


@pytest.mark.parametrize("devices", [None, "0,0"], ids=["one-gpu", "two-slabs"])
def test_reference_test_kernel_cpp_on_the_drop_in(devices):
    """The reference's own tests/test_kernel.cpp, unmodified, compiled against
    include/fdwave/kernel.hpp and linked to libfdwave_cuda.so (oracle/Makefile);
    also with every 3D Solver split into two Z slabs (FDW_DEVICES=0,0, the
    multi-GPU drop-in emulated on one GPU)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "test_kernel_cuda")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_kernel_cuda not built (needs the reference tree at build time)")
    env = dict(os.environ)
    if devices:
        env["FDW_DEVICES"] = devices
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
