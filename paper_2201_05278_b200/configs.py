"""Synthetic workloads C1-C5 of BASELINE.json / SURVEY.md section 8(d).

The velocity is deterministic (no RNG), defined on the interior grid (node
coincident, so resample_model is exact up to its interpolation weights):
    v = vmin + (vmax - vmin) * (iz / (nz - 1)) * (0.85 + 0.15 * (0.5 + 0.5 * sin(2 pi i_fast / n_fast)))
with the last element pinned to vmax, so c_max = vmax.  Damping alpha = 0.0015,
p = 3; Z-low null Neumann, every other face null Dirichlet; one 10 Hz Ricker at
half-cell offsets; receiver lines of 1700 (2D) / 800 (3D).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .acquisition import build_injection_map, make_point_set, ricker_wavelet
from .grid import Precision, build_grid, extend_with_damping
from .kernel import BoundaryCondition, BoundarySpec
from .model import damping_field, raw_planes_needed, resample_model
from .stencil import make_stencil
from .time_axis import build_time_axis

N, D = BoundaryCondition.NullNeumann, BoundaryCondition.NullDirichlet


@dataclass
class SyntheticConfig:
    name: str
    ndim: int
    bbox: list
    spacing: list
    space_order: int
    damping: list
    vmin: float
    vmax: float
    tf: float
    dt: Optional[float] = None
    alpha: float = 0.0015
    power: float = 3.0
    bc: list = field(default_factory=lambda: [[N, D], [D, D], [D, D]])
    f0: float = 10.0
    sources: list = field(default_factory=list)
    receivers: list = field(default_factory=list)
    window_radius: int = 4
    fixed_steps: Optional[int] = None  # C5: tf chosen so n_steps == fixed_steps

    def describe(self) -> dict:
        return {"name": self.name, "ndim": self.ndim, "space_order": self.space_order,
                "bbox": self.bbox, "spacing": self.spacing, "damping": self.damping}


def _rec_line_2d(n=1700):
    return [(25.0, 5.0 + 10.0 * k, 0.0) for k in range(n)]


def _rec_line_3d(n=800):
    return [(30.0, 10.0 + 20.0 * k, 8010.0) for k in range(n)]


def marmousi2d(order: int) -> SyntheticConfig:
    """C1 (SO2) / C2 (SO8): 351x1701 interior + 700 m damping -> 421x1841."""
    return SyntheticConfig(
        name=f"marmousi2d-so{order}", ndim=2, bbox=[0.0, 3500.0, 0.0, 17000.0], spacing=[10.0, 10.0],
        space_order=order, damping=[0.0, 700.0, 700.0, 700.0], vmin=1500.0, vmax=4700.0, tf=2.0,
        sources=[(45.0, 8505.0, 0.0)], receivers=_rec_line_2d())


def overthrust3d(order: int, z_planes_ext: int = 217) -> SyntheticConfig:
    """C3 (SO4) / C4 (SO8): 207x801x801 interior + 100 m damping -> 217x811x811.
    `z_planes_ext` = 217*P builds the weak-scaling grid with one Overthrust
    slab per GPU (interior Z = z_planes_ext - 10)."""
    nz_int = z_planes_ext - 10
    return SyntheticConfig(
        name=f"overthrust3d-so{order}" + ("" if z_planes_ext == 217 else f"-z{z_planes_ext}"),
        ndim=3, bbox=[0.0, 20.0 * (nz_int - 1), 0.0, 16000.0, 0.0, 16000.0], spacing=[20.0, 20.0, 20.0],
        space_order=order, damping=[100.0] * 6, vmin=2000.0, vmax=6000.0, tf=4.0,
        sources=[(50.0, 8010.0, 8010.0)], receivers=_rec_line_3d())


def weak3d(world: int, per_gpu: int = 200, steps: int = 500) -> SyntheticConfig:
    """C5: 200*P extended Z planes x 811 x 811, SO8, fixed 500 steps."""
    cfg = overthrust3d(8, z_planes_ext=per_gpu * world)
    cfg.name = f"weak3d-p{world}"
    cfg.fixed_steps = steps
    return cfg


CONFIGS = {
    "C1": lambda: marmousi2d(2),
    "C2": lambda: marmousi2d(8),
    "C3": lambda: overthrust3d(4),
    "C4": lambda: overthrust3d(8),
}


def synthetic_raw(shape, vmin: float, vmax: float, z_range=None) -> np.ndarray:
    """Raw interior velocity (double).  z_range restricts to raw Z planes."""
    nz = shape[0]
    nf = shape[-1]
    lo, hi = (0, nz) if z_range is None else z_range
    lat = np.array([0.85 + 0.15 * (0.5 + 0.5 * math.sin(2.0 * math.pi * i / nf)) for i in range(nf)])
    depth = np.array([float(iz) / float(nz - 1) for iz in range(lo, hi)])
    if len(shape) == 2:
        v = vmin + ((vmax - vmin) * depth[:, None]) * lat[None, :]
        if hi == nz:
            v[-1, -1] = vmax
        return np.ascontiguousarray(v)
    v = vmin + ((vmax - vmin) * depth[:, None, None]) * lat[None, None, :]
    v = np.broadcast_to(v, (hi - lo, shape[1], nf)).copy()
    if hi == nz:
        v[-1, -1, -1] = vmax
    return v


@dataclass
class Workload:
    cfg: SyntheticConfig
    grid: object
    axis: object
    coeffs: object
    spec: BoundarySpec
    velocity: np.ndarray  # padded (local slab for ranks)
    eta: np.ndarray
    sources: object
    wavelet: np.ndarray
    receivers: object
    c_max: float
    slab: Optional[tuple] = None  # (rank, world, z_begin, z_end)


def build_workload(cfg: SyntheticConfig, dtype=np.float32, rank: int = 0, world: int = 1,
                   with_fields: bool = True) -> Workload:
    """Runs the reference's setup chain (runner.hpp:42-110) on the synthetic
    model with the host mirror; for world > 1 only this rank's padded slab of
    the velocity/eta fields is built."""
    prec = Precision.Single if np.dtype(dtype) == np.float32 else Precision.Double
    g = build_grid(cfg.bbox, cfg.spacing[:cfg.ndim], cfg.space_order, prec)
    g = extend_with_damping(g, cfg.damping)
    raw_shape = tuple(g.interior_shape[:cfg.ndim])
    P = g.padded_shape()
    slab = None
    planes = None
    if world > 1:
        from ._lib import lib
        import ctypes as C
        zb, ze = C.c_uint64(), C.c_uint64()
        rc = lib().fdw_slab_range(g.extended_shape[0], world, rank, C.byref(zb), C.byref(ze))
        if rc != 0:
            raise ValueError(f"cannot split {g.extended_shape[0]} planes over {world} ranks")
        slab = (rank, world, zb.value, ze.value)
        planes = (zb.value, ze.value + 2 * g.halo)
    vel = eta = None
    if with_fields:
        if planes is None:
            raw = synthetic_raw(raw_shape, cfg.vmin, cfg.vmax)
            vel = resample_model(raw, raw_shape, g, dtype)
        else:
            rlo, rhi = raw_planes_needed(g, raw_shape[0], planes)
            rhi = min(rhi, raw_shape[0])
            raw = synthetic_raw(raw_shape, cfg.vmin, cfg.vmax, (rlo, rhi))
            vel = resample_model(raw, raw_shape, g, dtype, planes=planes, raw_z_offset=rlo)
        eta = damping_field(g, cfg.alpha, cfg.power, dtype, planes=planes).eta
    c_max = float(np.dtype(dtype).type(cfg.vmax))  # MaterialModel::c_max (pinned max)
    if cfg.fixed_steps is not None:
        from .stencil import stable_dt
        dt = stable_dt(c_max, g.spacing[:g.ndim], g.space_order, g.ndim)
        axis = build_time_axis(dt * cfg.fixed_steps, dt, 0, c_max, g)
    else:
        axis = build_time_axis(cfg.tf, cfg.dt, 0, c_max, g)
    src = build_injection_map(make_point_set(cfg.sources, cfg.window_radius), g)
    rec = build_injection_map(make_point_set(cfg.receivers, cfg.window_radius), g)
    wav = ricker_wavelet(axis, cfg.f0)
    spec = BoundarySpec([list(cfg.bc[a]) for a in range(3)])
    return Workload(cfg, g, axis, make_stencil(cfg.space_order), spec, vel, eta, src, wav, rec, c_max, slab)
