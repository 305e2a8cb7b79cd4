"""Reductions and the reference's partition API (drop-in for helmdef parallel.py).

``reduce_dot`` / ``reduce_norm`` run the library's deterministic device
reduction: fixed per-block partials combined in a fixed order, so the result
never depends on how the work is split (the contract of parallel.py:168-195).

The reference parallelises with host threads over a 2D tiling
(``partition_grid`` / ``WorkerPool`` / ``halo_exchange``, parallel.py:48-165).
On the GPU a level is one kernel launch, so the tiling does not drive the
compute here; the names are kept so reference callers run unchanged:
``partition_grid`` returns the same nested tiles (useful to callers that
inspect or post-process per tile), ``WorkerPool`` is a host thread pool with
the same ``run``/``close`` contract, ``halo_exchange`` returns the ghost-padded
snapshot as a ``PaddedField``.  ``LevelOperator.apply(u, out, pool, tiles)``
accepts and ignores pool/tiles (the device computes every tile at once).
The multi-GPU decomposition of this build is ``distributed.slab_plan``.
"""
from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import device as dev
from ._lib import check, lib

__all__ = ["Tile", "Partition", "WorkerPool", "partition_grid", "halo_exchange", "PaddedField", "reduce_dot",
           "reduce_norm", "HALO_RADII"]

# ghost rows each phase reads (radius-1 stencils, level-2 5x5, levels >= 3 7x7, transfers)
HALO_RADII = {"radius1": 1, "level2": 2, "coarse": 3, "transfer": 2}


def reduce_dot(u, v, pool=None) -> complex:
    """conj(u) . v (deterministic device reduction); pool is accepted and unused."""
    if tuple(u.shape) != tuple(v.shape):
        raise ValueError("reduce_dot needs identically shaped fields")
    du, dv = dev.to_device(u), dev.to_device(v)
    out = (C.c_double * 2)()
    check(lib().hdb_dot(du.data_ptr(), dv.data_ptr(), du.numel(), out))
    return complex(out[0], out[1])


def reduce_norm(u, pool=None) -> float:
    return float(np.sqrt(max(reduce_dot(u, u).real, 0.0)))


# ---------------------------------------------------------------- tiling (API)
@dataclass(frozen=True)
class Tile:
    """Rows [j0, j1) x columns [i0, i1) of one level."""

    j0: int
    j1: int
    i0: int
    i1: int

    @property
    def npoints(self) -> int:
        return (self.j1 - self.j0) * (self.i1 - self.i0)


@dataclass
class Partition:
    workers: int
    tiles: dict = field(default_factory=dict)          # level -> [Tile]
    halo_radius: dict = field(default_factory=lambda: dict(HALO_RADII))

    def level_tiles(self, level: int):
        return self.tiles[level]


def _cuts(n: int, parts: int, snap: int) -> list:
    """Interior cut positions of n into `parts` near-equal pieces, each rounded
    to the nearest multiple of `snap`; empty or repeated cuts are dropped."""
    out = []
    for t in range(1, parts):
        c = min(max(int(round(round(t * n / parts) / snap)) * snap, 0), n)
        if 0 < c < n and (not out or c > out[-1]):
            out.append(c)
    return out


def partition_grid(hierarchy, workers: int) -> Partition:
    """Nested near-square tiling for `workers` workers (parallel.py:71-109 contract):
    a x b = workers with the smallest ceil(ny/a) + ceil(nx/b); cut positions on the
    fine grid are multiples of 2**(ml-1), so level l's tiles are the fine cuts / 2**(l-1)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    fine = hierarchy.level(1)
    shapes = [(a, workers // a) for a in range(1, workers + 1) if workers % a == 0]
    rows_split, cols_split = min(shapes, key=lambda ab: -(-fine.ny // ab[0]) - (-fine.nx // ab[1]))
    snap = 1 << (hierarchy.ml - 1)
    ycut, xcut = _cuts(fine.ny, rows_split, snap), _cuts(fine.nx, cols_split, snap)
    part = Partition(workers=workers)
    for l in range(1, hierarchy.ml + 1):
        lv, s = hierarchy.level(l), 1 << (l - 1)
        ys = [0, *(c // s for c in ycut), lv.ny]
        xs = [0, *(c // s for c in xcut), lv.nx]
        part.tiles[l] = [Tile(y0, y1, x0, x1) for y0, y1 in zip(ys, ys[1:]) for x0, x1 in zip(xs, xs[1:])
                         if y1 > y0 and x1 > x0]
    return part


class WorkerPool:
    """Host thread pool with the reference's contract (parallel.py:112-139): run(fn,
    items) executes every item, inline for one worker, and re-raises the first
    exception; usable as a context manager."""

    def __init__(self, workers: int = 1):
        self.workers = max(1, int(workers))
        self._ex = ThreadPoolExecutor(max_workers=self.workers) if self.workers > 1 else None

    def run(self, fn, items):
        work = list(items)
        if self._ex is None or len(work) < 2:
            for it in work:
                fn(it)
            return
        for fut in [self._ex.submit(fn, it) for it in work]:
            fut.result()

    def close(self):
        if self._ex is not None:
            self._ex.shutdown(wait=True)
            self._ex = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass
class PaddedField:
    """Ghost-padded snapshot (radius r band) and per-tile windows into it."""

    data: np.ndarray
    radius: int

    def tile_window(self, tile: Tile) -> np.ndarray:
        r2 = 2 * self.radius
        return self.data[tile.j0:tile.j1 + r2, tile.i0:tile.i1 + r2]

    def interior(self) -> np.ndarray:
        r = self.radius
        return self.data[r:self.data.shape[0] - r, r:self.data.shape[1] - r]


def halo_exchange(u, pad_fn, radius: int) -> PaddedField:
    """Ghost snapshot for one stencil phase: pad_fn (e.g. LevelOperator.pad) applies
    the physical closure; interior tile halos are neighbours' values by construction."""
    return PaddedField(data=pad_fn(u), radius=radius)
