"""Off-grid sources/receivers and wavelets -- mirror of fdwave/acquisition.hpp
and the special functions it needs (special.hpp:49-71, :113-118).

InterpolationMap is held in CSR form (offsets, index, weight) -- the layout the
C-ABI consumes -- with `points` as the reference's list-of-lists view.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def bessel_i0(x: float) -> float:
    """special.hpp:49-71."""
    x = abs(x)
    if x < 100.0:
        q = 0.25 * x * x
        term, s = 1.0, 1.0
        for k in range(1, 200):
            term *= q / (float(k) * k)
            s += term
            if term < s * 1e-17:
                break
        return s
    term, s = 1.0, 1.0
    for k in range(1, 30):
        odd = 2.0 * k - 1.0
        term *= odd * odd / (8.0 * k * x)
        s += term
        if abs(term) < s * 1e-17:
            break
    return math.exp(x) / math.sqrt(2.0 * math.pi * x) * s


def sinc(x: float) -> float:
    """special.hpp:113-118: sin(pi x)/(pi x) with exact zeros at integers."""
    if x == math.floor(x):
        return 1.0 if x == 0.0 else 0.0
    px = math.pi * x
    if abs(px) < 1e-4:
        return 1.0 - px * px / 6.0
    return math.sin(px) / px


def kaiser_window(x: float, radius: int, b: float) -> float:
    """acquisition.hpp:21-27."""
    if radius < 1:
        raise ValueError("kaiser_window: radius must be >= 1")
    if not b > 0.0:
        raise ValueError("kaiser_window: b must be > 0")
    u = x / float(radius)
    if abs(u) > 1.0:
        return 0.0
    return bessel_i0(b * math.sqrt(1.0 - u * u)) / bessel_i0(b)


_KAISER_B = (1.24, 2.94, 4.53, 6.31, 7.91, 9.42, 10.88, 12.33, 13.80, 14.93)


def default_kaiser_b(radius: int) -> float:
    """acquisition.hpp:31-37 (Hicks 2002, Table 1)."""
    if radius < 1 or radius > 10:
        raise ValueError("window radius must be in [1, 10]")
    return _KAISER_B[radius - 1]


@dataclass
class HicksWeights:  # acquisition.hpp:42-45
    n_min: int = 0
    w: list = field(default_factory=list)


def hicks_weights_1d(alpha: float, radius: int, b: float) -> HicksWeights:
    """acquisition.hpp:47-59."""
    r = float(radius)
    n_lo = int(math.ceil(-r - alpha))
    n_hi = int(math.floor(r - alpha))
    hw = HicksWeights(n_min=n_lo)
    for n in range(n_lo, n_hi + 1):
        x = float(n) + alpha
        hw.w.append(kaiser_window(x, radius, b) * sinc(x))
    return hw


@dataclass
class PointSet:  # acquisition.hpp:62-66
    coordinates: list = field(default_factory=list)
    window_radius: int = 4
    kaiser_b: float = 6.31


def make_point_set(coordinates, window_radius: int = 4) -> PointSet:
    return PointSet(coordinates=[tuple(float(v) for v in c) for c in coordinates],
                    window_radius=window_radius, kaiser_b=default_kaiser_b(window_radius))


@dataclass
class InterpolationMap:  # acquisition.hpp:79-85, CSR
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    index: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    weight: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    @property
    def n_points(self) -> int:
        return len(self.offsets) - 1

    @property
    def points(self):
        return [list(zip(self.index[self.offsets[p]:self.offsets[p + 1]].tolist(),
                         self.weight[self.offsets[p]:self.offsets[p + 1]].tolist()))
                for p in range(self.n_points)]

    @staticmethod
    def from_points(points) -> "InterpolationMap":
        off = [0]
        idx, w = [], []
        for entries in points:
            for i, wt in entries:
                idx.append(int(i))
                w.append(float(wt))
            off.append(len(idx))
        return InterpolationMap(np.asarray(off, np.uint64), np.asarray(idx, np.uint64),
                                np.asarray(w, np.float64))


def build_injection_map(point_set: PointSet, grid) -> InterpolationMap:
    """acquisition.hpp:89-147: tensor product of per-axis windowed-sinc
    stencils; taps past the extended grid are dropped without renormalising."""
    if point_set.window_radius < 1 or point_set.window_radius > 10:
        raise ValueError("window radius must be in [1, 10]")
    P = grid.padded_shape()
    s0, s1 = P[1] * P[2], P[2]
    h = grid.halo
    ext = grid.extended_shape
    offs = [0]
    idx_parts, w_parts = [], []
    total = 0
    for coord in point_set.coordinates:
        aw = [None, None, None]
        nearest = [0, 0, 0]
        for a in range(grid.ndim):
            if coord[a] < grid.bbox[a][0] - 1e-9 or coord[a] > grid.bbox[a][1] + 1e-9:
                raise ValueError("point coordinate outside physical bounding box")
            pos = (coord[a] - grid.bbox[a][0]) / grid.spacing[a] + float(grid.damping_cells[a][0])
            nearest[a] = int(math.floor(pos + 0.5))
            alpha = float(nearest[a]) - pos
            aw[a] = hicks_weights_1d(alpha, point_set.window_radius, point_set.kaiser_b)
        if grid.ndim == 2:
            aw[2] = HicksWeights(0, [1.0])
            nearest[2] = 0
        iz = nearest[0] + aw[0].n_min + np.arange(len(aw[0].w))
        ix = nearest[1] + aw[1].n_min + np.arange(len(aw[1].w))
        iy = (nearest[2] + aw[2].n_min + np.arange(len(aw[2].w))) if grid.ndim == 3 else np.zeros(1, np.int64)
        wz = np.asarray(aw[0].w)
        wx = np.asarray(aw[1].w)
        wy = np.asarray(aw[2].w)
        w = (wz[:, None, None] * wx[None, :, None]) * wy[None, None, :]
        ok = ((iz >= 0) & (iz < ext[0]))[:, None, None] & ((ix >= 0) & (ix < ext[1]))[None, :, None]
        if grid.ndim == 3:
            ok = ok & ((iy >= 0) & (iy < ext[2]))[None, None, :]
        ok = ok & (w != 0.0)
        yoff = h if grid.ndim == 3 else 0
        flat = ((iz[:, None, None] + h) * s0 + (ix[None, :, None] + h) * s1 + (iy[None, None, :] + yoff))
        sel = np.broadcast_to(ok, w.shape)
        idx_parts.append(np.broadcast_to(flat, w.shape)[sel].astype(np.uint64))
        w_parts.append(w[sel])
        total += int(sel.sum())
        offs.append(total)
    if idx_parts:
        return InterpolationMap(np.asarray(offs, np.uint64), np.concatenate(idx_parts),
                                np.concatenate(w_parts))
    return InterpolationMap()


def sample_receivers(level: np.ndarray, imap: InterpolationMap) -> np.ndarray:
    """acquisition.hpp:150-161 on a host level (double accumulation per point,
    in entry order)."""
    flat = level.reshape(-1)
    out = np.empty(imap.n_points, level.dtype)
    for p in range(imap.n_points):
        acc = 0.0
        a, b = int(imap.offsets[p]), int(imap.offsets[p + 1])
        for i, w in zip(imap.index[a:b].tolist(), imap.weight[a:b].tolist()):
            acc += w * float(flat[i])
        out[p] = acc
    return out


def ricker_samples(count: int, dt: float, peak_frequency: float) -> np.ndarray:
    """acquisition.hpp:165-177, tau = t - 1/f."""
    if not peak_frequency > 0.0:
        raise ValueError("ricker: peak frequency must be > 0")
    t0 = 1.0 / peak_frequency
    s = np.empty(count, np.float64)
    pf = peak_frequency
    for n in range(count):
        tau = float(n) * dt - t0
        q = math.pi * math.pi * pf * pf * tau * tau
        s[n] = (1.0 - 2.0 * q) * math.exp(-q)
    return s


def ricker_wavelet(axis, peak_frequency: float) -> np.ndarray:
    """acquisition.hpp:179-181."""
    return ricker_samples(axis.sample_count(), axis.dt, peak_frequency)


def resample_wavelet(samples, axis) -> np.ndarray:
    """acquisition.hpp:185-199."""
    samples = [float(v) for v in samples]
    if len(samples) < 2:
        raise ValueError("wavelet file needs at least two samples")
    s = np.empty(axis.sample_count(), np.float64)
    scale = float(len(samples) - 1) / axis.tf
    for n in range(len(s)):
        pos = min(axis.time(n) * scale, float(len(samples) - 1))
        i = min(int(pos), len(samples) - 2)
        w = pos - float(i)
        s[n] = (1.0 - w) * samples[i] + w * samples[i + 1]
    return s
