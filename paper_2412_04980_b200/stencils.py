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
    h_power: int     # -2: Laplace-like (divided by h_l^2 when applied), 0: mass-like

    def __post_init__(self):
        side = len(self.numerators)
        if side % 2 == 0 or any(len(row) != side for row in self.numerators):
            raise ValueError("stencil must be square with odd side length")
        d = self.denominator
        if d <= 0 or d & (d - 1):
            raise ValueError("denominator must be a positive power of two")

    @property
    def radius(self) -> int:
        return len(self.numerators) // 2

    def as_array(self):
        import numpy as np
        return np.array(self.numerators, dtype=object)

    def as_float(self):
        import numpy as np
        return np.array(self.numerators, dtype=np.float64) / float(self.denominator)

    def is_symmetric(self) -> bool:
        """Invariant under transposition and both reflections (the D4 symmetry of the chain)."""
        rows = [list(r) for r in self.numerators]
        cols = [list(c) for c in zip(*rows)]
        return rows == cols and rows == rows[::-1] and rows == [r[::-1] for r in rows]

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


# ------------------------------------------------------------------ 2D coarsening
def _triple_matrix(radius_in: int):
    """Integer matrix T (7 x (2 r + 1)) of the 1D triple product: for a 1D stencil f
    with offsets -r..r, (T f)[d + 3] = sum_{a,s} w[a] f[s] w[a + s - 2d] (the same
    map `_triple_1d` applies)."""
    w = PROLONG_NUMERATORS_1D
    T = [[0] * (2 * radius_in + 1) for _ in range(7)]
    for d in range(-3, 4):
        for s in range(-radius_in, radius_in + 1):
            T[d + 3][s + radius_in] = sum(w[a + 2] * w[a + s - 2 * d + 2] for a in range(-2, 3)
                                          if -2 <= a + s - 2 * d <= 2)
    return T


def galerkin_coarsen(laplace: StencilKernel, mass: StencilKernel):
    """One exact Galerkin coarsening Z^T S Z of a 2D kernel pair (stencils.py:149-180
    contract).  The 2D triple product with the tensor transfer w (x) w factorises
    per axis, so each kernel becomes T S T^T with T the integer 1D triple-product
    matrix; the denominator gains 8**4 and is then reduced to canonical form.
    Works for any square integer kernel (not only separable ones); feeding
    level_kernels(l) returns level_kernels(l + 1)."""
    out = []
    for kern in (laplace, mass):
        S, r = kern.numerators, kern.radius
        T = _triple_matrix(r)
        TS = [[sum(T[p][q] * S[q][c] for q in range(2 * r + 1)) for c in range(2 * r + 1)] for p in range(7)]
        C = [[sum(TS[p][c] * T[k][c] for c in range(2 * r + 1)) for k in range(7)] for p in range(7)]
        table = {(x - 3, y - 3): C[y][x] for y in range(7) for x in range(7) if C[y][x]}
        rows, den = _canonical(table, kern.denominator * PROLONG_DENOMINATOR_1D ** 4)
        out.append(StencilKernel(rows, den, kern.h_power))
    return out[0], out[1]


@lru_cache(maxsize=1)
def _published_tables():
    """The paper's integer level 3-6 kernels (reference
    stencils.py:215-308), shipped as package data."""
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "data",
                           "published_kernel_tables.json")) as f:
        raw = json.load(f)
    return {int(l): {k: (tuple(tuple(r) for r in v[0]), int(v[1])) for k, v in d.items()} for l, d in raw.items()}


def __getattr__(name):  # REFERENCE_KERNELS is loaded lazily from the data file
    if name == "REFERENCE_KERNELS":
        return _published_tables()
    raise AttributeError(name)


def verify_chain(kernels=None):
    """Compare a kernel chain (default: level_kernels) with the published tables
    (stencils.py:321-371 contract).  One record per (level, kind) with keys level,
    kind, exact_match, within_ulp (entries beyond 2**53 may differ from the
    published float-derived values by <= 3 ulp) and first_mismatch
    ((row, col, derived, published), or (-1, -1, den, published den))."""
    import math
    provider = kernels if kernels is not None else level_kernels
    records = []
    for level, tabs in sorted(_published_tables().items()):
        for kind, kern in zip(("laplace", "mass"), provider(level)):
            want_rows, want_den = tabs[kind]
            exact = within = kern.denominator == want_den
            first = None
            for r, (got_row, want_row) in enumerate(zip(kern.numerators, want_rows)):
                for c, (got, want) in enumerate(zip(got_row, want_row)):
                    if got == want:
                        continue
                    exact = False
                    ulp = max(1, int(math.ulp(float(abs(got)))))
                    if abs(want) > 2 ** 53 and abs(got - want) <= 3 * ulp:
                        continue
                    within = False
                    first = first or (r, c, got, want)
            if kern.denominator != want_den:
                within = False
                first = first or (-1, -1, kern.denominator, want_den)
            records.append({"level": level, "kind": kind, "exact_match": exact, "within_ulp": within,
                            "first_mismatch": first})
    return records
