"""FD coefficients and CFL bound -- mirror of fdwave/stencil.hpp.

Pure-Python doubles in the reference's operation order (same Gaussian
elimination with partial pivoting), so the coefficients and dt are bit-identical.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


def _check_order(order: int) -> None:  # stencil.hpp:46-49
    if order < 2 or order > 20 or order % 2 != 0:
        raise ValueError("spatial order must be even and in [2, 20]")


def _solve_dense(a, b):  # stencil.hpp:17-44
    n = len(b)
    a = [list(r) for r in a]
    b = list(b)
    for col in range(n):
        pivot = col
        for row in range(col + 1, n):
            if abs(a[row][col]) > abs(a[pivot][col]):
                pivot = row
        a[col], a[pivot] = a[pivot], a[col]
        b[col], b[pivot] = b[pivot], b[col]
        if a[col][col] == 0.0:
            raise RuntimeError("singular stencil moment system")
        for row in range(col + 1, n):
            f = a[row][col] / a[col][col]
            if f == 0.0:
                continue
            for k in range(col, n):
                a[row][k] -= f * a[col][k]
            b[row] -= f * b[col]
    x = [0.0] * n
    for row in range(n - 1, -1, -1):
        s = b[row]
        for k in range(row + 1, n):
            s -= a[row][k] * x[k]
        x[row] = s / a[row][row]
    return x


def second_derivative_coefficients(order: int) -> list:
    """stencil.hpp:55-72: v_0..v_r."""
    _check_order(order)
    r = order // 2
    a = [[0.0] * r for _ in range(r)]
    rhs = [0.0] * r
    for m in range(1, r + 1):
        inv_fact = 1.0
        for k in range(2, 2 * m + 1):
            inv_fact /= float(k)
        for j in range(1, r + 1):
            a[m - 1][j - 1] = math.pow(float(j), float(2 * m)) * inv_fact
        rhs[m - 1] = inv_fact if m == 1 else 0.0
    v = _solve_dense(a, rhs)
    s = 0.0
    for c in v:
        s += c
    return [-2.0 * s] + v


def first_derivative_coefficients(order: int) -> list:
    """stencil.hpp:77-90: w_1..w_r."""
    _check_order(order)
    r = order // 2
    a = [[0.0] * r for _ in range(r)]
    rhs = [0.0] * r
    for m in range(1, r + 1):
        inv_fact = 1.0
        for k in range(2, 2 * m):
            inv_fact /= float(k)
        for j in range(1, r + 1):
            a[m - 1][j - 1] = math.pow(float(j), float(2 * m - 1)) * inv_fact
        rhs[m - 1] = inv_fact if m == 1 else 0.0
    return _solve_dense(a, rhs)


@dataclass
class StencilCoeffs:  # stencil.hpp:93-98
    order: int = 2
    radius: int = 1
    second: list = field(default_factory=list)
    first: list = field(default_factory=list)


def make_stencil(order: int) -> StencilCoeffs:
    """stencil.hpp:100-107."""
    return StencilCoeffs(order=order, radius=order // 2,
                         second=second_derivative_coefficients(order),
                         first=first_derivative_coefficients(order))


def stable_dt(c_max: float, spacing, order: int, ndim: int) -> float:
    """stencil.hpp:113-129: dt = 2 dx_min / (c_max sqrt(ndim (|v0| + 2 sum|vj|)))."""
    if c_max <= 0.0:
        raise ValueError("stable_dt: c_max must be > 0")
    if ndim not in (2, 3):
        raise ValueError("stable_dt: ndim must be 2 or 3")
    if len(spacing) == 0:
        raise ValueError("stable_dt: empty spacing")
    dx_min = float(spacing[0])
    for h in spacing:
        if h <= 0.0:
            raise ValueError("stable_dt: spacing must be > 0")
        dx_min = min(dx_min, float(h))
    v = second_derivative_coefficients(order)
    abs_sum = abs(v[0])
    for j in range(1, len(v)):
        abs_sum += 2.0 * abs(v[j])
    a = float(ndim) * abs_sum
    return 2.0 * dx_min / (c_max * math.sqrt(a))
