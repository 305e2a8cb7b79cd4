"""Vertex-centred hierarchy and benchmark problems (oracle restatement).

Restates grid.py:184-195 (wedge layer rule), grid.py:220-294 (build_hierarchy:
point counts, coarsenability, k^2 = (2 pi f / c)^2 on level 1, injection
ksq[::2, ::2] below), grid.py:309-320 (point source 1/(hx*hy) at the nearest
node) and grid.py:381-413 (mp1 / wedge problem builders).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SOMMERFELD = "sommerfeld"
DIRICHLET = "dirichlet"

REFERENCE_WEDGE = [(-400.0, -500.0, 2000.0), (-800.0, -600.0, 1500.0), (0.0, 0.0, 3000.0)]
# BASELINE.json configs[2] geometry (interfaces (0,400)->(600,200), (0,800)->(600,600) m depth)
BASELINE_WEDGE = [(-400.0, -200.0, 2000.0), (-800.0, -600.0, 1500.0), (0.0, 0.0, 3000.0)]
WEDGE_DOMAIN = ((0.0, 600.0), (-1000.0, 0.0))


@dataclass(frozen=True)
class Level:
    level: int
    nx: int
    ny: int
    h: float
    origin: tuple

    @property
    def npoints(self):
        return self.nx * self.ny

    @property
    def shape(self):
        return (self.ny, self.nx)


@dataclass
class Hierarchy:
    levels: list
    ksq: list
    boundary: tuple

    @property
    def ml(self):
        return len(self.levels)

    def level(self, l):
        return self.levels[l - 1]

    def ksq_at(self, l):
        return self.ksq[l - 1]

    @property
    def extent(self):
        lv = self.levels[0]
        return (lv.h * (lv.nx - 1), lv.h * (lv.ny - 1))


def _npts(length, h):
    n = length / h
    if abs(n - round(n)) > 1e-8 * max(1.0, abs(n)):
        raise ValueError(f"extent {length} not a multiple of {h}")
    return int(round(n)) + 1


def wedge_speed(layers, x, y):
    """Top-down layer assignment, last layer catch-all (grid.py:184-195)."""
    xx, yy = np.meshgrid(x, y)
    lx = x[-1] - x[0] if x.size > 1 else 1.0
    c = np.full(xx.shape, layers[-1][2], dtype=np.float64)
    free = np.ones(xx.shape, dtype=bool)
    for ya, yb, v in layers[:-1]:
        surf = ya + (yb - ya) * (xx - x[0]) / lx
        sel = free & (yy >= surf)
        c[sel] = v
        free &= ~sel
    return c


def build_hierarchy(domain, h, ml, *, k=None, layers=None, f=None, speed=None,
                    boundary=SOMMERFELD) -> Hierarchy:
    """grid.py:220-287.  Exactly one of k (constant), layers (+f) or speed
    (a callable (x, y) -> c array, + f) defines k^2 on level 1."""
    (x0, x1), (y0, y1) = domain
    nx, ny = _npts(x1 - x0, h), _npts(y1 - y0, h)
    step = 2 ** (ml - 1)
    if ml < 2 or (nx - 1) % step or (ny - 1) % step:
        raise ValueError(f"{nx}x{ny} cannot be coarsened {ml - 1} times")
    bnd = (boundary,) * 4 if isinstance(boundary, str) else tuple(boundary)
    levels, ksq = [], []
    cx, cy, ch = nx, ny, float(h)
    for l in range(1, ml + 1):
        levels.append(Level(l, cx, cy, ch, (x0, y0)))
        if l == 1:
            xs = x0 + ch * np.arange(cx)
            ys = y0 + ch * np.arange(cy)
            if k is not None:
                kk = np.full((cy, cx), float(k) ** 2)
            else:
                c = wedge_speed(layers, xs, ys) if layers is not None else speed(xs, ys)
                kk = (2.0 * math.pi * f / c) ** 2
        else:
            kk = ksq[-1][::2, ::2].copy()
        ksq.append(np.ascontiguousarray(kk))
        cx, cy, ch = (cx - 1) // 2 + 1, (cy - 1) // 2 + 1, 2.0 * ch
    return Hierarchy(levels, ksq, bnd)


def point_source(hier: Hierarchy, loc) -> np.ndarray:
    """grid.py:309-320: 1/(h*h) at the nearest node, returned as (ny, nx)."""
    lv = hier.level(1)
    i = int(round((loc[0] - lv.origin[0]) / lv.h))
    j = int(round((loc[1] - lv.origin[1]) / lv.h))
    b = np.zeros(lv.shape, dtype=np.complex128)
    b[j, i] = 1.0 / (lv.h * lv.h)
    return b


def mp1_problem(k, n, ml, boundary=SOMMERFELD):
    """grid.py:381-398 with n given: unit square, h = 1/(n-1), centre source."""
    hier = build_hierarchy(((0.0, 1.0), (0.0, 1.0)), 1.0 / (n - 1), ml, k=k, boundary=boundary)
    return hier, point_source(hier, (0.5, 0.5))


def wedge_problem(f, nx, ml, layers=REFERENCE_WEDGE):
    """grid.py:401-413 with nx given; source at (300, 0)."""
    h = 600.0 / (nx - 1)
    hier = build_hierarchy(WEDGE_DOMAIN, h, ml, layers=layers, f=f)
    return hier, point_source(hier, (300.0, 0.0))


def baseline_wedge_problem(f, h=0.5, ml=5):
    """BASELINE configs[2]: BASELINE geometry on the reference wedge domain."""
    hier = build_hierarchy(WEDGE_DOMAIN, h, ml, layers=BASELINE_WEDGE, f=f)
    return hier, point_source(hier, (300.0, 0.0))
