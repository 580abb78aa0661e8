"""Caller integration: the reference's own run driver
(config.hpp parse_run_config -> runner.hpp run_simulation -> io.hpp writers:
seismogram CSV / raw+sidecar, snapshot raw+sidecar and PGM, manifest) built
against the drop-in (integration/_build/fdwave_cuda) must write the SAME
bytes as the same driver on the reference's CPU Solver
(integration/_build/fdwave_cpu), for strided snapshots, variable density and
both precisions; plus the bench / verify / coeff subcommands on the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")


def _exe(name):
    p = os.path.join(BUILD, name)
    if not os.path.exists(p):
        pytest.skip(f"integration/_build/{name} not built (needs the reference tree at build time)")
    return p


def _model(d, name, arr, units):
    arr.astype(np.float32).tofile(os.path.join(d, name + ".bin"))
    with open(os.path.join(d, name + ".json"), "w") as f:
        json.dump({"shape": list(arr.shape), "dtype": "f32", "units": units}, f)
    return {"path": os.path.join(d, name + ".bin"), "sidecar": os.path.join(d, name + ".json")}


def _config(d, ndim, dtype, stride, density, dt=None, rec_z=25.0):
    if ndim == 2:
        shape, bbox, h = (41, 61), [0, 400, 0, 600], [10.0, 10.0]
        src, recs = [[45.0, 305.0]], [[25.0, 15.0 + 20.0 * k] for k in range(25)]
        bc = ["null_neumann", "null_dirichlet", "null_dirichlet", "null_dirichlet"]
        damping = [0, 100, 100, 100]
    else:
        shape, bbox, h = (21, 31, 26), [0, 200, 0, 300, 0, 250], [10.0, 10.0, 10.0]
        src, recs = [[45.0, 155.0, 125.0]], [[rec_z, 15.0 + 20.0 * k, 125.0] for k in range(12)]
        bc = ["null_neumann", "null_dirichlet", "null_dirichlet", "null_dirichlet", "none", "null_dirichlet"]
        damping = [0, 50, 50, 50, 50, 50]
    iz = np.arange(shape[0]).reshape((-1,) + (1,) * (ndim - 1))
    vel = 1500.0 + 2500.0 * iz / (shape[0] - 1) + 0.0 * np.zeros(shape)
    cfg = {
        "bounding_box": bbox, "grid_spacing": h, "space_order": 8, "dtype": dtype,
        "velocity_model": _model(d, "vel", vel, "m/s"),
        "boundary": {"damping_length": damping, "boundary_condition": bc, "damping_polynomial_degree": 3,
                     "damping_alpha": 0.002},
        "time": {"tf": 0.25, "saving_stride": stride},
        "sources": {"coordinates": src, "window_radius": 4},
        "receivers": {"coordinates": recs, "window_radius": 4},
        "wavelet": {"type": "ricker", "peak_frequency": 15.0},
        "backend": {"type": "parallel", "workers": 0},
    }
    if dt is not None:
        cfg["time"]["dt"] = dt
    if density:
        rho = 1.0 + 1.5 * iz / (shape[0] - 1) + 0.0 * np.zeros(shape)
        rho[shape[0] // 2:] += 0.4
        cfg["density_model"] = _model(d, "rho", rho, "g/cm3")
    p = os.path.join(d, "config.json")
    with open(p, "w") as f:
        json.dump(cfg, f)
    return p


def _run(exe, cfg, out):
    return subprocess.run([exe, "run", "--config", cfg, "--out", out], capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("ndim,dtype,stride,density", [
    (2, "float32", 10, False), (2, "float64", 7, True), (3, "float32", 25, True), (3, "float64", 0, False)])
def test_run_artifacts_identical_to_the_cpu_reference(tmp_path, ndim, dtype, stride, density):
    cfg = _config(str(tmp_path), ndim, dtype, stride, density)
    outs = {}
    for name in ("fdwave_cpu", "fdwave_cuda"):
        out = str(tmp_path / name)
        r = _run(_exe(name), cfg, out)
        assert r.returncode == 0, r.stderr
        outs[name] = out
    a, b = outs["fdwave_cpu"], outs["fdwave_cuda"]
    files = sorted(os.listdir(a))
    assert files == sorted(os.listdir(b))
    n_snap = sum(f.endswith(".pgm") for f in files)
    assert n_snap >= (2 if stride else 1)
    for f in files:
        if f == "manifest.json":
            ma, mb = json.load(open(os.path.join(a, f))), json.load(open(os.path.join(b, f)))
            ma.pop("kernel_seconds"), mb.pop("kernel_seconds")
            assert ma == mb
        else:
            assert open(os.path.join(a, f), "rb").read() == open(os.path.join(b, f), "rb").read(), f


@pytest.mark.parametrize("devices,dtype,stride,density,rec_z", [
    ("0,0", "float32", 25, True, 25.0), ("0,0,0", "float64", 0, False, 25.0), ("0,0", "float32", 0, False, 125.0),
    ("0,0,0", "float64", 20, False, 95.0)])
def test_run_on_slabs_identical_to_the_cpu_reference(tmp_path, devices, dtype, stride, density, rec_z):
    """The reference's unmodified runner.hpp `Solver<T> solver(...)` spread over
    several GPUs (FDW_DEVICES: Z slabs, halo planes over peer memory), here
    emulated on one GPU: every artefact must still be byte-identical to the CPU
    reference -- also with the receiver line across a slab face (rec_z 125 m /
    95 m: taps on two slabs, merged from per-tap products in entry order)."""
    cfg = _config(str(tmp_path), 3, dtype, stride, density, rec_z=rec_z)
    a = str(tmp_path / "cpu")
    assert _run(_exe("fdwave_cpu"), cfg, a).returncode == 0
    b = str(tmp_path / "cuda")
    r = subprocess.run([_exe("fdwave_cuda"), "run", "--config", cfg, "--out", b], capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, FDW_DEVICES=devices))
    assert r.returncode == 0, r.stderr
    files = sorted(os.listdir(a))
    assert files == sorted(os.listdir(b))
    for f in files:
        if f == "manifest.json":
            ma, mb = json.load(open(os.path.join(a, f))), json.load(open(os.path.join(b, f)))
            ma.pop("kernel_seconds"), mb.pop("kernel_seconds")
            assert ma == mb
        else:
            assert open(os.path.join(a, f), "rb").read() == open(os.path.join(b, f), "rb").read(), f


@pytest.mark.parametrize("ndim", [2, 3])
def test_run_verbose_progress_matches_the_cpu_reference(tmp_path, ndim):
    """`run --verbose` (runner.hpp:84 set_verbose): the reference prints
    "step s/N  t s  max|p| = m" at every health check (kernel.hpp:459-466).
    The drop-in must print the same lines -- same steps, same max|p| digits --
    with only the elapsed time differing."""
    import re
    cfg = _config(str(tmp_path), ndim, "float32", 0, False)
    pat = re.compile(r"^step (\d+)/(\d+)  (\d+\.\d{3})s  max\|p\| = (\S+)$")
    got = {}
    for name in ("fdwave_cpu", "fdwave_cuda"):
        r = subprocess.run([_exe(name), "run", "--config", cfg, "--out", str(tmp_path / name), "--verbose"],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        lines = [m.groups() for m in (pat.match(l) for l in r.stderr.splitlines()) if m]
        assert lines, r.stderr
        got[name] = [(a, b, d) for a, b, _, d in lines]
    assert got["fdwave_cuda"] == got["fdwave_cpu"]
    assert got["fdwave_cpu"][-1][0] == got["fdwave_cpu"][-1][1]  # the last step is checked


def test_run_instability_exit_code(tmp_path):
    cfg = _config(str(tmp_path), 2, "float32", 0, False, dt=5e-3)  # far above the CFL bound
    for name in ("fdwave_cpu", "fdwave_cuda"):
        r = _run(_exe(name), cfg, str(tmp_path / name))
        assert r.returncode == 2, (name, r.stdout, r.stderr)
        assert "numerical failure" in r.stderr


def test_run_accepts_a_cuda_backend(tmp_path):
    cfg = _config(str(tmp_path), 2, "float32", 0, False)
    j = json.load(open(cfg))
    j["backend"] = {"type": "cuda", "workers": 0}
    json.dump(j, open(cfg, "w"))
    r = _run(_exe("fdwave_cuda"), cfg, str(tmp_path / "o"))
    assert r.returncode == 0, r.stderr


def test_bench_subcommand_on_the_gpu(tmp_path):
    csv = str(tmp_path / "bench.csv")
    r = subprocess.run([_exe("fdwave_cuda"), "bench", "--grid", "96,96,96", "--orders", "2,8", "--steps", "60",
                        "--repetitions", "2", "--emit-csv", csv], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "backend equivalence probe" in r.stdout and "[pass]" in r.stdout
    rows = open(csv).read().strip().splitlines()
    assert len(rows) == 1 + 4  # 2 orders x (serial, parallel)


def test_verify_subcommand_analytical_gate_on_the_gpu():
    r = subprocess.run([_exe("fdwave_cuda"), "verify", "analytical"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[pass]" in r.stdout


def test_coeff_subcommand():
    r = subprocess.run([_exe("fdwave_cuda"), "coeff", "--order", "4"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0
    vals = [float(x) for x in r.stdout.split()]
    assert vals == pytest.approx([-2.5, 4 / 3, -1 / 12], rel=1e-15)
