"""Exact-integer Galerkin stencil chain (oracle restatement).

Restates stencils.py:101-196 (level-1 pair, triple product with the
(1,4,6,4,1) transfer numerators, power-of-two reduction, level_kernels) in a
different but exactly equivalent form: every level-l kernel is a sum of
tensor products of 1D integer factors, so the 2D triple product is
computed as 1D triple products followed by outer products.  The 2D integer
tables this produces are compared against the reference's published tables
(stencils.py:215-308, dumped to tests/golden/kernel_tables.json).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

W = (1, 4, 6, 4, 1)          # stencils.py:39-42 transfer numerators
TRANSFER_DEN_2D_SQ = 64 * 64  # (8*8)^2, stencils.py:149-160


def _coarsen_1d(f: dict) -> dict:
    """1D Galerkin triple product  c(d) = sum_a sum_s w(a) f(s) w(a+s-2d)."""
    out = {}
    for d in range(-3, 4):
        acc = 0
        for a in range(-2, 3):
            for s, fv in f.items():
                e = a + s - 2 * d
                if -2 <= e <= 2:
                    acc += W[a + 2] * fv * W[e + 2]
        out[d] = acc
    return out


def _outer(p: dict, q: dict) -> dict:
    """2D table t[(dx, dy)] = p[dx] * q[dy]."""
    return {(dx, dy): pv * qv for dx, pv in p.items() for dy, qv in q.items()}


def _add(*tabs) -> dict:
    out = {}
    for t in tabs:
        for k, v in t.items():
            out[k] = out.get(k, 0) + v
    return out


def _to_table(entries: dict, den: int):
    """Power-of-two reduction (stencils.py:142-146) + radius crop (stencils.py:162-176)."""
    while den % 2 == 0 and all(v % 2 == 0 for v in entries.values()):
        entries = {k: v // 2 for k, v in entries.items()}
        den //= 2
    nz = [max(abs(dx), abs(dy)) for (dx, dy), v in entries.items() if v != 0]
    r = max(max(nz, default=1), 1)
    n = 2 * r + 1
    tab = [[0] * n for _ in range(n)]
    for (dx, dy), v in entries.items():
        if abs(dx) <= r and abs(dy) <= r:
            tab[dy + r][dx + r] = v
    return tab, den, r


@lru_cache(maxsize=None)
def _factors(level: int):
    """1D factors (a, m) with  lap_l = a(x)m + m(x)a,  mass_l = m(x)m  (unreduced)."""
    if level == 1:
        return {-1: -1, 0: 2, 1: -1}, {0: 1}
    a, m = _factors(level - 1)
    return _coarsen_1d(a), _coarsen_1d(m)


@lru_cache(maxsize=None)
def level_kernels(level: int):
    """(lap_table, lap_den, mass_table, mass_den, radius) — exact ints.

    Same values as stencils.level_kernels (stencils.py:183-196).  The
    denominators accumulate (8*8)^2 per level before reduction, exactly as
    galerkin_coarsen does (stencils.py:159-160); reduction is applied to the
    accumulated 2D table at every level (same canonical form).
    """
    if level == 1:
        return ((0, -1, 0), (-1, 4, -1), (0, -1, 0)), 1, ((0, 0, 0), (0, 1, 0), (0, 0, 0)), 1, 1
    lap_prev, lden, mass_prev, mden, _ = level_kernels(level - 1)
    outs = []
    for tab, den in ((lap_prev, lden), (mass_prev, mden)):
        r = len(tab) // 2
        # decompose the previous 2D table into rows of 1D coarsenings:
        # coarsen(T)(dx,dy) = sum_{sx,sy} T[sy][sx] * c1(sx->dx) c1(sy->dy)
        entries = {}
        for sy in range(-r, r + 1):
            for sx in range(-r, r + 1):
                v = tab[sy + r][sx + r]
                if v == 0:
                    continue
                cx = _coarsen_1d({sx: 1})
                cy = _coarsen_1d({sy: 1})
                for (dx, dy), pv in _outer(cx, cy).items():
                    if pv:
                        entries[(dx, dy)] = entries.get((dx, dy), 0) + v * pv
        for d in ((dx, dy) for dx in range(-3, 4) for dy in range(-3, 4)):
            entries.setdefault(d, 0)
        t, dn, rad = _to_table(entries, den * TRANSFER_DEN_2D_SQ)
        outs.append((tuple(tuple(row) for row in t), dn, rad))
    (lt, ld, lr), (mt, md, mr) = outs
    assert lr == mr
    return lt, ld, mt, md, lr


def mass_level_scale(level: int) -> float:
    """4**(level-1)  (stencils.py:199-201)."""
    return float(4 ** (level - 1))


def separable_factors(level: int):
    """Float 1D factors for the separable apply (used only by tests that
    check the product's separable coefficients).  Returns (a, m, lap_c, mass_c)
    with lap_table == lap_c * (a(x)m + m(x)a), mass_table == mass_c * m(x)m."""
    a, m = _factors(level)
    lt, ld, mt, md, r = level_kernels(level)
    lap2 = _add(_outer(a, m), _outer(m, a))
    mass2 = _outer(m, m)
    ratios = []
    for tab, ref in ((lt, lap2), (mt, mass2)):
        from fractions import Fraction
        rr = None
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                v = tab[dy + r][dx + r]
                w_ = ref.get((dx, dy), 0)
                if w_ != 0:
                    q = Fraction(v, w_)
                    assert rr is None or rr == q
                    rr = q
                else:
                    assert v == 0
        ratios.append(rr)
    av = np.array([a.get(d, 0) for d in range(-r, r + 1)], dtype=np.float64)
    mv = np.array([m.get(d, 0) for d in range(-r, r + 1)], dtype=np.float64)
    return av, mv, ratios[0], ratios[1]


def verify_against_tables(tables: dict):
    """Compare derived tables with reference tables {level: {kind: (rows, den)}}.

    Exact equality below 2**53; above, within 3 ulp (the reference's own
    tolerance for its float-rounded level-6 mass entries, stencils.py:310-319).
    """
    import math
    bad = []
    for level, kinds in tables.items():
        lt, ld, mt, md, _ = level_kernels(int(level))
        for kind, (rows, den) in kinds.items():
            got, gden = (lt, ld) if kind == "laplace" else (mt, md)
            if gden != den:
                bad.append((level, kind, "den", gden, den))
            for r in range(len(rows)):
                for c in range(len(rows)):
                    g, w_ = got[r][c], rows[r][c]
                    if g == w_:
                        continue
                    if abs(w_) > 2 ** 53 and abs(g - w_) <= 3 * max(1, int(math.ulp(float(abs(g))))):
                        continue
                    bad.append((level, kind, r, c, g, w_))
    return bad
