"""Seeded synthetic velocity models and benchmark-problem builders (host setup).

`synthetic_layered_velocity` is BASELINE configs[3]'s model, which the
reference does not ship (its `synthetic_marmousi_velocity`,
grid.py:350-378, is an unseeded stand-in): a 9192 m x 3000 m raster of ~30
sinusoidally folded layers whose velocity increases with depth (1500-5500 m/s),
cut by 4 random dipping faults that offset the layers by 50-200 m, then
smoothed with a Gaussian of sigma = 2 cells.  Everything is drawn from
numpy's default_rng(seed), so the same seed gives the same raster on any
host; the raster is consumed through VelocityModel(kind="gridfile") by this
package and by the reference alike (bilinear sampling, grid.py:198-217).
"""
from __future__ import annotations

import math

import numpy as np

from .grid import Problem, VelocityModel, build_hierarchy, point_source_device, point_source_rhs

__all__ = ["synthetic_layered_velocity", "synthetic_layered_problem", "C4_DOMAIN", "C4_SOURCE", "c5_problem"]

C4_DOMAIN = ((0.0, 9192.0), (-3000.0, 0.0))
C4_SOURCE = (4596.0, 0.0)


def _gauss_smooth(a: np.ndarray, sigma: float) -> np.ndarray:
    """Separable Gaussian filter, reflect padding, radius 4 sigma."""
    r = int(math.ceil(4 * sigma))
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    w /= w.sum()
    out = a
    for axis in (0, 1):
        pad = [(0, 0), (0, 0)]
        pad[axis] = (r, r)
        p = np.pad(out, pad, mode="reflect")
        acc = np.zeros_like(out)
        for k, wk in enumerate(w):
            sl = [slice(None), slice(None)]
            sl[axis] = slice(k, k + out.shape[axis])
            acc += wk * p[tuple(sl)]
        out = acc
    return out


def synthetic_layered_velocity(seed: int = 2412, dx: float = 6.0, n_layers: int = 30, n_faults: int = 4,
                               vmin: float = 1500.0, vmax: float = 5500.0, sigma_cells: float = 2.0) -> VelocityModel:
    (x0, x1), (y0, y1) = C4_DOMAIN
    rng = np.random.default_rng(seed)
    nxv = int(round((x1 - x0) / dx)) + 1
    nyv = int(round((y1 - y0) / dx)) + 1
    xs = x0 + dx * np.arange(nxv)
    depth = (y1 - (y0 + dx * np.arange(nyv)))[:, None]  # 0 at the surface, positive downward
    X = np.broadcast_to(xs[None, :], (nyv, nxv))
    D = np.broadcast_to(depth, (nyv, nxv)).copy()
    # faults: a dipping line through (xf, 0); the hanging wall (x beyond the trace) drops by `throw`
    for _ in range(n_faults):
        xf = rng.uniform(0.1, 0.9) * (x1 - x0) + x0
        dip = math.radians(rng.uniform(50.0, 80.0)) * rng.choice([-1.0, 1.0])
        throw = rng.uniform(50.0, 200.0)
        trace = xf + D / math.tan(dip)
        D = np.where(X > trace, D - throw, D)
    # folded interfaces: base depth + sum of two sinusoids
    base = np.sort(rng.uniform(0.0, 1.0, n_layers - 1)) * (y1 - y0) * 1.05
    layer = np.zeros((nyv, nxv), dtype=np.int64)
    for i, zb in enumerate(base):
        a1, a2 = rng.uniform(20.0, 120.0), rng.uniform(5.0, 40.0)
        l1, l2 = rng.uniform(2000.0, 8000.0), rng.uniform(600.0, 2000.0)
        p1, p2 = rng.uniform(0, 2 * math.pi, 2)
        surf = zb + a1 * np.sin(2 * math.pi * xs / l1 + p1) + a2 * np.sin(2 * math.pi * xs / l2 + p2)
        layer += (D >= surf[None, :]).astype(np.int64)
    trend = np.linspace(vmin, vmax, n_layers)
    v_layer = np.clip(trend + rng.uniform(-150.0, 150.0, n_layers), vmin, vmax)
    v_layer[0] = vmin
    vel = v_layer[np.clip(layer, 0, n_layers - 1)]
    vel = np.clip(_gauss_smooth(vel, sigma_cells), vmin, vmax)
    # rows already run from y0 = -3000 m (row 0) up to the surface, as the grid does
    return VelocityModel(kind="gridfile", values=np.ascontiguousarray(vel), dx=dx, dy=dx, x0=x0, y0=y0)


def synthetic_layered_problem(f: float, h: float, ml: int, seed: int = 2412, raster_dx: float = 6.0,
                              device: bool = False) -> Problem:
    """BASELINE configs[3]: the seeded model at mesh width h (9192 = 2^3 3 383 m, so h = 24/2^p
    and ml <= p + 1), point source at (4596, 0) m, Sommerfeld on all sides."""
    vel = synthetic_layered_velocity(seed, dx=raster_dx)
    hier = build_hierarchy(C4_DOMAIN, h=h, ml=ml, velocity=vel, f=f, boundary="sommerfeld", device=device)
    rhs = point_source_device(hier, C4_SOURCE) if device else point_source_rhs(hier, C4_SOURCE)
    return Problem("synthetic-layered", hier, rhs)


def c5_problem(P: int = 1, ml: int = 7, device: bool = False, cells: int = 8192) -> Problem:
    """BASELINE configs[4] (weak scaling): [0,1] x [0,P], h = 1/8192 (8193 x (8192P+1) points,
    SURVEY D8), k = (0.5 / h^2)^(1/3) so that k^3 h^2 = 0.5, centre source, Sommerfeld.
    `cells` per unit length scales the instance down (the parity fixture uses 1024, P = 2)."""
    h = 1.0 / cells
    k = (0.5 / h ** 2) ** (1.0 / 3.0)
    hier = build_hierarchy(((0.0, 1.0), (0.0, float(P))), h=h, ml=ml, k=k, boundary="sommerfeld", device=device)
    rhs = point_source_device(hier, (0.5, P / 2.0)) if device else point_source_rhs(hier, (0.5, P / 2.0))
    return Problem("c5", hier, rhs)
