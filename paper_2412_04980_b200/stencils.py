"""Exact-rational level kernels (setup only; host integer arithmetic).

Every level kernel of the Galerkin chain (reference stencils.py:101-196) is a
sum of tensor products of two 1D integer factors,

    laplace_l = a_l (x) m_l + m_l (x) a_l,      mass_l = m_l (x) m_l,

with a_1 = (-1, 2, -1), m_1 = (0, 1, 0) and each coarsening the 1D triple
product with the (1, 4, 6, 4, 1) transfer numerators.  This module derives the
1D chain, forms the 2D integer tables over the accumulated power-of-two
denominator 4096**(l-1), and reduces them to canonical form.  The result is
checked against the reference's published tables in tests (exact below 2**53).

The float conversion used by the kernels (operators.py:111-113) happens in
``operators.LevelOperator``.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

PROLONG_NUMERATORS_1D = (1, 4, 6, 4, 1)
PROLONG_DENOMINATOR_1D = 8
RESTRICT_DENOMINATOR_1D = 16
TRANSFER_ADJOINT_SCALE = 4.0


@dataclass(frozen=True)
class StencilKernel:
    """Square integer stencil over a power-of-two denominator."""

    numerators: tuple
    denominator: int
    h_power: int

    @property
    def radius(self) -> int:
        return len(self.numerators) // 2

    def as_float(self):
        import numpy as np
        return np.array(self.numerators, dtype=np.float64) / float(self.denominator)

    def coefficient_sum(self):
        return sum(sum(r) for r in self.numerators)


def _triple_1d(f):
    """c[d] = sum_{a,s} w[a] f[s] w[a + s - 2d]  over offsets a, a+s-2d in [-2, 2]."""
    w = PROLONG_NUMERATORS_1D
    out = [0] * 7  # d = -3..3
    for d in range(-3, 4):
        tot = 0
        for s, fv in f.items():
            if fv == 0:
                continue
            for a in range(-2, 3):
                e = a + s - 2 * d
                if -2 <= e <= 2:
                    tot += w[a + 2] * w[e + 2] * fv
        out[d + 3] = tot
    return {d - 3: v for d, v in enumerate(out)}


@lru_cache(maxsize=None)
def factors_1d(level: int):
    """Unreduced 1D factors (a_l, m_l) as {offset: int}."""
    if level < 1:
        raise ValueError("level must be >= 1")
    if level == 1:
        return {-1: -1, 0: 2, 1: -1}, {-1: 0, 0: 1, 1: 0}
    a, m = factors_1d(level - 1)
    return _triple_1d(a), _triple_1d(m)


def _canonical(table: dict, den: int):
    while den % 2 == 0 and all(v % 2 == 0 for v in table.values()):
        table = {k: v // 2 for k, v in table.items()}
        den //= 2
    radius = max([max(abs(x), abs(y)) for (x, y), v in table.items() if v] or [1])
    radius = max(radius, 1)
    rows = tuple(tuple(table.get((x, y), 0) for x in range(-radius, radius + 1))
                 for y in range(-radius, radius + 1))
    return rows, den


@lru_cache(maxsize=None)
def level_kernels(level: int):
    """(laplace, mass) StencilKernel pair of a level (1 = finest)."""
    a, m = factors_1d(level)
    den = 4096 ** (level - 1)
    lap = {}
    mass = {}
    for x, ax in a.items():
        for y, my in m.items():
            lap[(x, y)] = lap.get((x, y), 0) + ax * my
            lap[(y, x)] = lap.get((y, x), 0) + ax * my
    for x, mx in m.items():
        for y, my in m.items():
            mass[(x, y)] = mx * my
    lrows, lden = _canonical(lap, den)
    mrows, mden = _canonical(mass, den)
    # both kernels of a level share the radius of the wider one
    r = max(len(lrows), len(mrows)) // 2
    lrows, mrows = _pad(lrows, r), _pad(mrows, r)
    return (StencilKernel(lrows, lden, -2), StencilKernel(mrows, mden, 0))


def _pad(rows, r):
    cur = len(rows) // 2
    if cur == r:
        return rows
    n = 2 * r + 1
    d = r - cur
    out = [[0] * n for _ in range(n)]
    for y, row in enumerate(rows):
        for x, v in enumerate(row):
            out[y + d][x + d] = v
    return tuple(tuple(r_) for r_ in out)


def mass_level_scale(level: int) -> float:
    """4**(level-1): value normalisation carried by the mass chain."""
    return float(4 ** (level - 1))
