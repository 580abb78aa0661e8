"""Volume sources (ModulatedField, kernel.hpp:140-144, :199-203, :439-452) on
the CUDA path against the oracle, bit-exact; and the reference's verification
harness (verify.hpp) run through the drop-in header on the GPU:
  * oracle/_ref/test_verify_cuda -- the reference's tests/test_verify.cpp;
  * oracle/_ref/verify_cuda      -- analytical agreement case + MMS / temporal /
    spatial convergence studies; the errors must equal the CPU reference's
    (tests/golden/verify_ref_quick.jsonl, written by oracle/_ref/verify_ref
    from the same driver, tests/cpp/verify_cuda.cpp) digit for digit."""
import json
import os
import subprocess

import numpy as np
import pytest

from helpers import D, N, X, same, small_config
import oracle as O
from paper_2201_05278_b200 import DampingField, ModulatedField, Solver, make_material_model
from paper_2201_05278_b200._lib import FDW_KERNEL_SIMPLE, FDW_KERNEL_TMA, FDW_KERNEL_ZMARCH
from paper_2201_05278_b200.configs import build_workload

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFBIN = os.path.join(ROOT, "oracle", "_ref")


def _fields(shape, dtype, steps, seed):
    rng = np.random.default_rng(seed)
    f1 = (rng.standard_normal(shape) * 1e-3).astype(dtype)
    f2 = np.zeros(shape, dtype)
    f2[tuple(slice(s // 3, 2 * s // 3) for s in shape)] = 2e-3
    a1 = np.sin(np.arange(steps + 5) * 0.21)
    a2 = np.cos(np.arange(steps) * 0.13) * 10.0
    return (f1, a1), (f2, a2)


@pytest.mark.parametrize("ndim,variant", [(2, 0), (2, FDW_KERNEL_SIMPLE), (3, 0), (3, FDW_KERNEL_SIMPLE),
                                          (3, FDW_KERNEL_ZMARCH), (3, FDW_KERNEL_TMA)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("with_density", [False, True])
def test_volume_sources_forward(ndim, variant, dtype, with_density):
    shape = (37, 45) if ndim == 2 else (21, 25, 23)
    cfg = small_config(ndim=ndim, order=8, shape=shape, bc=[[N, D], [D, X], [D, N]])
    w = build_workload(cfg, dtype)
    rho = None
    if with_density:
        rho = (1.5 + np.random.default_rng(2).random(w.velocity.shape)).astype(dtype)
    vols = _fields(w.velocity.shape, dtype, w.axis.n_steps, 7)
    g = Solver(w.grid, make_material_model(w.velocity, rho), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
               variant=variant)
    o = O.OracleSolver(ndim, 8, dtype, w.grid.extended_shape, w.grid.spacing, w.axis.dt, w.axis.n_steps,
                       w.spec.face, w.velocity, w.eta, density=rho)
    for s_ in (g, o):
        s_.set_sources(w.sources, w.wavelet)
        s_.set_receivers(w.receivers)
    for f, a in vols:
        g.add_volume_source(ModulatedField(field=f, amplitude=list(a)))
        o.add_volume_source(f, a)
    res = g.forward()
    ref = o.forward()
    assert np.abs(ref["final"]).max() > 0
    assert same(res.seismogram.data, ref["seismogram"])
    assert same(res.snapshots[-1], ref["final"])


def test_volume_source_rejects_short_amplitude():
    cfg = small_config(ndim=2, order=4, shape=(17, 19))
    w = build_workload(cfg, np.float32)
    g = Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs)
    with pytest.raises(ValueError):
        g.add_volume_source(ModulatedField(field=np.zeros(w.velocity.shape, np.float32),
                                           amplitude=[0.0] * (w.axis.n_steps - 1)))


def _need(name):
    exe = os.path.join(REFBIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"oracle/_ref/{name} not built (needs the reference tree at build time)")
    return exe


def test_reference_test_verify_cpp_on_the_drop_in():
    r = subprocess.run([_need("test_verify_cuda")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


def _reports(lines):
    return {d["study"]: d for d in (json.loads(l) for l in lines if l.strip().startswith("{"))}


def test_verification_harness_matches_the_cpu_reference():
    exe = _need("verify_cuda")
    r = subprocess.run([exe, "analytical", "mms", "temporal", "spatial", "quick"], capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stderr[-2000:]
    got = _reports(r.stdout.splitlines())
    # tools/main.cpp:123: the analytical agreement gate is 1 %
    assert got["analytical"]["relative_error"] <= 0.01
    with open(os.path.join(ROOT, "tests", "golden", "verify_ref_quick.jsonl")) as fh:
        want = _reports(fh.read().splitlines())
    for study, ref in want.items():
        assert got[study]["points"] == ref["points"], study  # identical traces -> identical errors
        assert got[study]["slope"] == ref["slope"], study
