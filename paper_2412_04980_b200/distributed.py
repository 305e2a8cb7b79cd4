"""Row-slab decomposition of the MADP solve over several ranks.

Grid depth d (d = 0 the finest grid, every deflation level and multigrid
sub-level sits at some depth) has ny_d = (ny - 1) / 2**d + 1 rows.  Depths
0..D-1 are SHARDED in row slabs whose fine cut rows are multiples of 2**(D-1),
so the slab of depth d is exactly the injection of the slab of depth d-1 (the
nesting rule of the reference's tiler, parallel.py:59-68,92-105, in 1D); D is
the largest depth count for which every rank keeps >= min_rows rows.  Deeper
depths are REPLICATED: every rank holds the whole (small) grid and computes it
redundantly and deterministically, entered by an all-gather of the restricted
slabs and left by a local prolongation, so no scatter is needed.

Transport: NCCL when each rank is a process with its own GPU
(`DistContext.nccl`), or host threads of one process (`DistContext.threads`,
one engine and stream per thread; kernels never wait on each other), which
runs the same slab code on a single GPU for testing.
"""
from __future__ import annotations

import ctypes as C
import itertools
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib

__all__ = ["SlabPlan", "slab_plan", "gather_rows", "DistContext"]

HALO = 3  # rows carried by vectors of sharded levels (max stencil radius)


@dataclass(frozen=True)
class SlabSpec:
    row0: int
    ny: int
    halo: int
    table_row0: tuple
    table_ny: tuple


@dataclass
class SlabPlan:
    ranks: int
    depths: int            # D: number of sharded depths
    snap: int              # fine cut rows are multiples of snap = 2**(D-1)
    cuts: list             # fine cut rows (ranks + 1 entries)
    ny0: int               # finest rows

    def rows_at(self, depth):
        return (self.ny0 - 1) // 2 ** depth + 1

    def sharded(self, depth) -> bool:
        return self.ranks > 1 and depth < self.depths

    def slab(self, depth, rank):
        """(row0, ny) of `rank` at `depth` (sharded depths only)."""
        s = 2 ** depth
        r0 = self.cuts[rank] // s
        r1 = self.cuts[rank + 1] // s if rank < self.ranks - 1 else self.rows_at(depth)
        return r0, r1 - r0

    def spec(self, depth, rank):
        if not self.sharded(depth):
            return None
        table = [self.slab(depth, r) for r in range(self.ranks)]
        r0, n = table[rank]
        return SlabSpec(r0, n, HALO, tuple(t[0] for t in table), tuple(t[1] for t in table))


def slab_plan(ny: int, ranks: int, max_depth: int, min_rows: int = 32) -> SlabPlan:
    """Largest nested slab partition of a grid with `ny` rows (coarsenable
    max_depth-1 times) where every rank keeps >= min_rows rows at every sharded depth."""
    if ranks < 1:
        raise ValueError("ranks must be >= 1")
    if ranks == 1:
        return SlabPlan(1, 0, 1, [0, ny], ny)
    for D in range(max_depth, 0, -1):
        snap = 2 ** (D - 1)
        if (ny - 1) % snap:
            continue
        units = (ny - 1) // snap
        base, extra = divmod(units, ranks)
        if base == 0:
            continue
        cuts = [0]
        for r in range(ranks):
            cuts.append(cuts[-1] + (base + (1 if r < extra else 0)) * snap)
        plan = SlabPlan(ranks, D, snap, cuts, ny)
        ok = all(plan.slab(D - 1, r)[1] >= min_rows for r in range(ranks))
        if ok:
            return plan
    return SlabPlan(ranks, 0, 1, [0, ny], ny)  # nothing sharded: every rank replicates


def gather_rows(plan: "SlabPlan", depth: int, rank: int):
    """(row0, ny): the rows of depth `depth + 1` this rank restricts and all-gathers
    when `depth` is the last sharded depth -- the library's own rule
    (hdb_plan_gather_rows; no device needed)."""
    from ._lib import load_library
    L = load_library()
    starts = (C.c_int * plan.ranks)(*[plan.slab(depth, r)[0] for r in range(plan.ranks)])
    r0, n = C.c_int(), C.c_int()
    check(L.hdb_plan_gather_rows(starts, plan.ranks, rank, plan.rows_at(depth + 1), C.byref(r0), C.byref(n)))
    return r0.value, n.value


_groups = itertools.count(1)


@dataclass
class DistContext:
    """This rank's place in the decomposition; binds the library's communicator."""

    rank: int
    size: int
    kind: str = "nccl"      # "nccl" | "threads"
    group: int = 0
    min_rows: int = 32
    _bound: bool = field(default=False, repr=False)

    @classmethod
    def nccl(cls, rank=None, size=None):
        """One process per GPU; torch.distributed must be initialised (any backend)."""
        import torch
        import torch.distributed as dist
        rank = dist.get_rank() if rank is None else rank
        size = dist.get_world_size() if size is None else size
        L = lib()
        uid = C.create_string_buffer(128)
        if rank == 0:
            check(L.hdb_comm_unique_id(uid))
        t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0)
        raw = bytes(t.cpu().numpy().tolist())
        check(L.hdb_comm_init_nccl(raw, size, rank))
        return cls(rank, size, "nccl", 0, _bound=True)

    @classmethod
    def threads(cls, rank, size, group, device=0):
        """Rank `rank` of `size` host threads sharing `group` (call inside the thread)."""
        L = lib()
        check(L.hdb_thread_engine_begin(device))
        check(L.hdb_comm_init_threads(group, size, rank))
        return cls(rank, size, "threads", group, _bound=True)

    @staticmethod
    def new_group() -> int:
        return next(_groups)

    def close(self):
        if self.kind == "threads" and self._bound:
            lib().hdb_thread_engine_end()
            self._bound = False
