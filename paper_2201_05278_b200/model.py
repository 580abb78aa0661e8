"""Material model and absorbing layer -- mirror of fdwave/model.hpp.

Vectorised with numpy in the reference's operation order (elementwise IEEE
double ops, no contraction), so the padded fields are bit-identical to the
reference's.  `planes=(lo, hi)` restricts a 3D field to padded Z planes
[lo, hi) -- the local slab of a multi-GPU rank -- without building the rest.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np


def _dtype(precision_or_dtype):
    return np.dtype(precision_or_dtype)


def _axis_weights(coord: float, lo: float, hi: float, raw_n: int):
    """model.hpp:21-26."""
    pos = (coord - lo) / (hi - lo) * float(raw_n - 1)
    clamped = 0.0 if pos < 0.0 else pos
    if float(raw_n - 1) < clamped:
        clamped = float(raw_n - 1)
    i0 = int(clamped)
    if raw_n - 2 < i0:
        i0 = raw_n - 2
    return i0, clamped - float(i0)


def _axis_table(grid, a: int, raw_n: int, n_pad: int):
    h = grid.halo
    lo = h + grid.damping_cells[a][0]
    n_int = grid.interior_shape[a]
    i0 = np.empty(n_pad, np.int64)
    w = np.empty(n_pad, np.float64)
    for p in range(n_pad):
        c = min(max(p, lo), lo + n_int - 1) - lo
        i0[p], w[p] = _axis_weights(grid.bbox[a][0] + float(c) * grid.spacing[a], grid.bbox[a][0],
                                    grid.bbox[a][1], raw_n)
    return i0, w


def resample_model(raw, raw_shape, grid, dtype=np.float32, planes=None, raw_z_offset=0) -> np.ndarray:
    """model.hpp:34-106: multilinear resample with edge replication into the
    ABL and halo.  Returns the padded field (Z, X[, Y]) of `dtype`.

    For a slab (`planes`), `raw` may hold only raw Z planes
    [raw_z_offset, raw_z_offset + raw.shape[0]) of the full raw_shape."""
    raw_shape = tuple(int(n) for n in raw_shape)
    if len(raw_shape) != grid.ndim:
        raise ValueError("resample_model: dimension mismatch with grid")
    if any(n < 2 for n in raw_shape):
        raise ValueError("resample_model: raw shape must be >= 2 per axis")
    raw = np.asarray(raw, dtype=np.float64)
    if raw_z_offset == 0 and raw.size == int(np.prod(raw_shape)):
        raw = raw.reshape(raw_shape)
    P = grid.padded_shape()
    z0, wz = _axis_table(grid, 0, raw_shape[0], P[0])
    x0, wx = _axis_table(grid, 1, raw_shape[1], P[1])
    lo, hi = (0, P[0]) if planes is None else planes
    dt = _dtype(dtype)
    if grid.ndim == 2:
        zz, ww = z0[lo:hi, None] - raw_z_offset, wz[lo:hi, None]
        xx, vx = x0[None, :], wx[None, :]
        value = (1 - ww) * ((1 - vx) * raw[zz, xx] + vx * raw[zz, xx + 1]) + \
            ww * ((1 - vx) * raw[zz + 1, xx] + vx * raw[zz + 1, xx + 1])
        return value.astype(dt)
    y0, wy = _axis_table(grid, 2, raw_shape[2], P[2])
    out = np.empty((hi - lo, P[1], P[2]), dt)
    X0, WX = x0[:, None], wx[:, None]
    Y0, WY = y0[None, :], wy[None, :]
    for k, pz in enumerate(range(lo, hi)):
        zi, zw = int(z0[pz]) - raw_z_offset, float(wz[pz])
        r0, r1 = raw[zi], raw[zi + 1]
        c00 = (1 - WY) * r0[X0, Y0] + WY * r0[X0, Y0 + 1]
        c01 = (1 - WY) * r0[X0 + 1, Y0] + WY * r0[X0 + 1, Y0 + 1]
        c10 = (1 - WY) * r1[X0, Y0] + WY * r1[X0, Y0 + 1]
        c11 = (1 - WY) * r1[X0 + 1, Y0] + WY * r1[X0 + 1, Y0 + 1]
        out[k] = (1 - zw) * ((1 - WX) * c00 + WX * c01) + zw * ((1 - WX) * c10 + WX * c11)
    return out


def raw_planes_needed(grid, raw_n0: int, planes) -> tuple:
    """Raw Z index range [lo, hi) that resample_model reads for padded planes."""
    z0, _ = _axis_table(grid, 0, raw_n0, grid.padded_shape()[0])
    sel = z0[planes[0]:planes[1]]
    return int(sel.min()), int(sel.max()) + 2


@dataclass
class MaterialModel:  # model.hpp:110-114
    velocity: np.ndarray
    density: Optional[np.ndarray] = None
    c_max: float = 0.0


def make_material_model(velocity: np.ndarray, density: Optional[np.ndarray] = None) -> MaterialModel:
    """model.hpp:116-137."""
    v = np.asarray(velocity)
    if not np.all(v > 0):
        raise ValueError("material model: velocity must be > 0 everywhere")
    if density is not None:
        if density.size != v.size:
            raise ValueError("material model: density shape mismatch")
        if not np.all(density > 0):
            raise ValueError("material model: density must be > 0 everywhere")
    return MaterialModel(velocity=v, density=density, c_max=float(v.max()))


@dataclass
class DampingField:  # model.hpp:141-146
    eta: np.ndarray
    alpha: float = 0.0
    power: float = 0.0


def _excess(grid, axis: int, n_pad: int) -> np.ndarray:
    """model.hpp:162-170: metres beyond the physical box along one axis."""
    out = np.zeros(n_pad, np.float64)
    for p in range(n_pad):
        rel = p - grid.halo - grid.damping_cells[axis][0]
        if rel < 0:
            out[p] = float(-rel) * grid.spacing[axis]
        elif rel >= grid.interior_shape[axis]:
            out[p] = float(rel - grid.interior_shape[axis] + 1) * grid.spacing[axis]
    return out


def damping_field(grid, alpha: float, power: float, dtype=np.float32, planes=None) -> DampingField:
    """model.hpp:148-186: eta = alpha * d^power, d the Euclidean distance to
    the physical box (zero inside).  pow() is evaluated with libm on the few
    distinct distances, exactly as the reference evaluates it per point."""
    if alpha < 0.0 or power < 0.0:
        raise ValueError("damping_field: alpha and power must be >= 0")
    P = grid.padded_shape()
    dt = _dtype(dtype)
    ez = _excess(grid, 0, P[0])
    ex = _excess(grid, 1, P[1])
    ey = _excess(grid, 2, P[2]) if grid.ndim == 3 else np.zeros(1)
    lo, hi = (0, P[0]) if planes is None else planes
    ez = ez[lo:hi]
    # distinct excess values per axis -> table of eta over the index triple
    uz, iz = np.unique(ez, return_inverse=True)
    ux, ix = np.unique(ex, return_inverse=True)
    uy, iy = np.unique(ey, return_inverse=True)
    table = np.zeros((len(uz), len(ux), len(uy)), dt)
    for a, dz in enumerate(uz):
        for b, dx in enumerate(ux):
            for c, dy in enumerate(uy):
                d = math.sqrt(dz * dz + dx * dx + dy * dy)
                table[a, b, c] = dt.type(alpha * math.pow(d, power)) if d > 0.0 else dt.type(0)
    if grid.ndim == 2:
        eta = table[iz[:, None], ix[None, :], 0]
    else:
        eta = table[iz[:, None, None], ix[None, :, None], iy[None, None, :]]
    return DampingField(eta=np.ascontiguousarray(eta), alpha=alpha, power=power)
