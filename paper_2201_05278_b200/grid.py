"""Grid geometry -- host mirror of /root/reference/proj/include/fdwave/grid.hpp.

Axis order is fixed: Z (depth) first, then X, then Y (grid.hpp:14-17).  The
extended shape is physical domain + absorbing-layer cells; the halo is tracked
separately and never counts as grid points.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field, replace


class Precision(enum.IntEnum):  # grid.hpp:12
    Single = 0
    Double = 1


def llround(x: float) -> int:
    """C llround: half away from zero."""
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


@dataclass
class Grid:  # grid.hpp:18-48
    ndim: int = 2
    bbox: list = field(default_factory=lambda: [[0.0, 0.0], [0.0, 0.0], [0.0, 0.0]])
    spacing: list = field(default_factory=lambda: [1.0, 1.0, 1.0])
    interior_shape: list = field(default_factory=lambda: [1, 1, 1])
    damping_cells: list = field(default_factory=lambda: [[0, 0], [0, 0], [0, 0]])
    damping_length: list = field(default_factory=lambda: [[0.0, 0.0], [0.0, 0.0], [0.0, 0.0]])
    halo: int = 1
    space_order: int = 2
    precision: Precision = Precision.Double
    extended_shape: list = field(default_factory=lambda: [1, 1, 1])

    def interior_points(self) -> int:
        return self.interior_shape[0] * self.interior_shape[1] * self.interior_shape[2]

    def extended_points(self) -> int:
        return self.extended_shape[0] * self.extended_shape[1] * self.extended_shape[2]

    def padded_shape(self) -> tuple:
        """grid.hpp:37-42: extended grid plus halo on every side of each axis."""
        p = [1, 1, 1]
        for a in range(self.ndim):
            p[a] = self.extended_shape[a] + 2 * self.halo
        return tuple(p)

    def node_coordinate(self, axis: int, i: int) -> float:
        low = float(self.damping_cells[axis][0])
        return self.bbox[axis][0] + (float(i) - low) * self.spacing[axis]

    def copy(self) -> "Grid":
        return replace(self, bbox=[list(b) for b in self.bbox], spacing=list(self.spacing),
                       interior_shape=list(self.interior_shape),
                       damping_cells=[list(d) for d in self.damping_cells],
                       damping_length=[list(d) for d in self.damping_length],
                       extended_shape=list(self.extended_shape))


def build_grid(bbox, spacing, space_order: int, precision: Precision = Precision.Single) -> Grid:
    """grid.hpp:50-80."""
    if len(bbox) not in (4, 6):
        raise ValueError("build_grid: bounding box needs 4 or 6 entries")
    ndim = len(bbox) // 2
    if len(spacing) != ndim:
        raise ValueError("build_grid: spacing must have one entry per axis")
    if space_order < 2 or space_order > 20 or space_order % 2 != 0:
        raise ValueError("build_grid: space order must be even in [2, 20]")
    g = Grid(ndim=ndim, space_order=space_order, halo=space_order // 2, precision=precision)
    for a in range(ndim):
        lo, hi = float(bbox[2 * a]), float(bbox[2 * a + 1])
        if not hi > lo:
            raise ValueError(f"build_grid: bbox max must exceed min (axis {a})")
        if not float(spacing[a]) > 0.0:
            raise ValueError(f"build_grid: spacing must be positive (axis {a})")
        g.bbox[a] = [lo, hi]
        g.spacing[a] = float(spacing[a])
        g.interior_shape[a] = llround((hi - lo) / g.spacing[a]) + 1
    g.extended_shape = list(g.interior_shape)
    return g


def extend_with_damping(grid: Grid, lengths) -> Grid:
    """grid.hpp:85-104: lengths are Zlo, Zhi, Xlo, Xhi[, Ylo, Yhi] in meters."""
    if len(lengths) != 2 * grid.ndim:
        raise ValueError("extend_with_damping: need two lengths per axis")
    g = grid.copy()
    for a in range(g.ndim):
        for side in range(2):
            ln = float(lengths[2 * a + side])
            if ln < 0.0:
                raise ValueError("extend_with_damping: damping length must be >= 0")
            g.damping_length[a][side] = ln
            g.damping_cells[a][side] = llround(ln / g.spacing[a])
        g.extended_shape[a] = g.interior_shape[a] + g.damping_cells[a][0] + g.damping_cells[a][1]
    return g
