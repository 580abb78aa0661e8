"""Shared builders for the parity tests (test code, not product code)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

import oracle as O
from paper_2201_05278_b200 import DampingField, Solver, make_material_model
from paper_2201_05278_b200.configs import SyntheticConfig, build_workload
from paper_2201_05278_b200.kernel import BoundaryCondition as BC

D, N, X = BC.NullDirichlet, BC.NullNeumann, BC.None_


def small_config(ndim=3, order=8, shape=(19, 29, 23), damping_cells=5, h=20.0, steps=None, bc=None,
                 n_rec=12, tf=None, src=None):
    """Synthetic case with the given INTERIOR shape (Z, X[, Y])."""
    bbox = []
    for n in shape[:ndim]:
        bbox += [0.0, h * (n - 1)]
    damping = [h * damping_cells] * (2 * ndim)
    if bc is None:
        bc = [[N, D], [D, D], [D, D]]
    mid = [h * (n - 1) / 2 + h / 2 for n in shape[:ndim]]
    if src is None:
        src = [(h * 2.5, mid[1], mid[2] if ndim == 3 else 0.0)]
    recs = [(h * 1.5, h * (0.5 + k * (shape[1] - 2) / max(n_rec, 1)), mid[2] if ndim == 3 else 0.0)
            for k in range(n_rec)]
    cfg = SyntheticConfig(name="small", ndim=ndim, bbox=bbox, spacing=[h] * ndim, space_order=order,
                          damping=damping, vmin=2000.0, vmax=6000.0, tf=tf or 0.1, sources=src,
                          receivers=recs, bc=bc, f0=12.0)
    if steps is not None:
        cfg.fixed_steps = steps
    return cfg


def gpu_solver(w, **kw):
    return Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
                  **kw)


def oracle_solver(w, threads=0):
    return O.OracleSolver(w.grid.ndim, w.grid.space_order, w.velocity.dtype, w.grid.extended_shape,
                          w.grid.spacing, w.axis.dt, w.axis.n_steps, w.spec.face, w.velocity, w.eta,
                          threads=threads)


def run_both(cfg, dtype=np.float32, **kw):
    w = build_workload(cfg, dtype)
    g = gpu_solver(w, **kw)
    g.set_sources(w.sources, w.wavelet)
    g.set_receivers(w.receivers)
    res = g.forward()
    o = oracle_solver(w)
    o.set_sources(w.sources, w.wavelet)
    o.set_receivers(w.receivers)
    ref = o.forward()
    return w, g, res, o, ref


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def same(a, b):
    """IEEE equality (signed zeros compare equal; NaN == NaN)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN_DIR) if f.endswith(".npz") and not f.startswith("full_"))


def load_golden(name):
    """(SyntheticConfig, dtype, meta, seismogram, final) of a committed fixture."""
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    meta = json.loads(str(z["meta"]))
    c = dict(meta["cfg"])
    c["sources"] = [tuple(p) for p in c["sources"]]
    c["receivers"] = [tuple(p) for p in c["receivers"]]
    cfg = SyntheticConfig(**c)
    return cfg, np.dtype(meta["dtype"]), meta, z["seismogram"], z["final"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
