"""Reductions and the row-slab partition (drop-in for reference parallel.py).

``reduce_dot`` / ``reduce_norm`` run the library's deterministic device
reduction (fixed grid, fixed-order partial combination: the result does not
depend on how the work is split, the contract of parallel.py:168-195).

``partition_slabs`` is the multi-GPU decomposition of this build: the finest
grid is cut into row slabs whose boundaries are multiples of 2**(D-1), D the
deepest sharded level, so every coarse level's slab is the injection of the
fine one (the nesting rule of parallel.py:59-68,92-105, in 1D).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import device as dev
from ._lib import check, lib

__all__ = ["reduce_dot", "reduce_norm", "Slab", "SlabPartition", "partition_slabs"]


def reduce_dot(u, v, pool=None) -> complex:
    """conj(u) . v (deterministic device reduction)."""
    if tuple(u.shape) != tuple(v.shape):
        raise ValueError("reduce_dot needs identically shaped fields")
    du, dv = dev.to_device(u), dev.to_device(v)
    out = (C.c_double * 2)()
    check(lib().hdb_dot(du.data_ptr(), dv.data_ptr(), du.numel(), out))
    return complex(out[0], out[1])


def reduce_norm(u, pool=None) -> float:
    return float(np.sqrt(max(reduce_dot(u, u).real, 0.0)))


@dataclass(frozen=True)
class Slab:
    rank: int
    j0: int  # first owned row (level-local)
    j1: int  # one past the last owned row

    @property
    def rows(self):
        return self.j1 - self.j0


@dataclass
class SlabPartition:
    ranks: int
    snap: int
    slabs: dict = field(default_factory=dict)  # level -> [Slab per rank]

    def level_slabs(self, level):
        return self.slabs[level]


def partition_slabs(hierarchy, ranks: int, sharded_levels: int | None = None) -> SlabPartition:
    """Row slabs of every level for ``ranks`` GPUs.

    Fine-grid split rows are multiples of snap = 2**(D-1) (D = number of
    sharded levels, default all), balanced to within one snap unit; the last
    rank also owns the final vertex row.  Level-l slab rows are the fine
    split rows divided by 2**(l-1), so restriction/prolongation between
    sharded levels never crosses a slab boundary by more than the transfer halo.
    """
    if ranks < 1:
        raise ValueError("ranks must be >= 1")
    D = hierarchy.ml if sharded_levels is None else sharded_levels
    snap = 2 ** (D - 1)
    ny = hierarchy.level(1).ny
    units = (ny - 1) // snap  # row intervals in snap units
    base, extra = divmod(units, ranks)
    cuts = [0]
    for r in range(ranks):
        cuts.append(cuts[-1] + (base + (1 if r < extra else 0)) * snap)
    part = SlabPartition(ranks=ranks, snap=snap)
    for l in range(1, hierarchy.ml + 1):
        scale = 2 ** (l - 1)
        nyl = hierarchy.level(l).ny
        if l <= D:
            rows = [c // scale for c in cuts]
            rows[-1] = nyl
            part.slabs[l] = [Slab(r, rows[r], rows[r + 1]) for r in range(ranks)]
        else:  # gathered level: rank 0 owns everything
            part.slabs[l] = [Slab(0, 0, nyl)] + [Slab(r, nyl, nyl) for r in range(1, ranks)]
    return part
