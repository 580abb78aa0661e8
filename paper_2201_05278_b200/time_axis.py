"""Time axis -- mirror of fdwave/time_axis.hpp."""
from __future__ import annotations

import math
from dataclasses import dataclass

from .stencil import stable_dt


@dataclass
class TimeAxis:  # time_axis.hpp:16-29
    tf: float = 0.0
    dt: float = 0.0
    n_steps: int = 0
    saving_stride: int = 0
    stable_bound: float = 0.0
    dt_overridden: bool = False

    def time(self, n: int) -> float:
        return float(n) * self.dt

    def sample_count(self) -> int:
        return self.n_steps + 1

    def snapshot_count(self) -> int:
        return 1 if self.saving_stride == 0 else self.n_steps // self.saving_stride + 1


def build_time_axis(tf: float, dt, saving_stride: int, c_max: float, grid) -> TimeAxis:
    """time_axis.hpp:31-50; dt None selects the CFL bound."""
    if not tf > 0.0:
        raise ValueError("build_time_axis: tf must be > 0")
    if dt is not None and not dt > 0.0:
        raise ValueError("build_time_axis: dt must be > 0")
    ax = TimeAxis(tf=float(tf))
    ax.stable_bound = stable_dt(c_max, grid.spacing[:grid.ndim], grid.space_order, grid.ndim)
    ax.dt = float(dt) if dt is not None else ax.stable_bound
    ax.dt_overridden = ax.dt > ax.stable_bound * (1.0 + 1e-12)
    ax.n_steps = int(math.ceil(tf / ax.dt * (1.0 - 1e-12)))
    if ax.n_steps == 0:
        ax.n_steps = 1
    ax.saving_stride = min(int(saving_stride), ax.n_steps)
    return ax
