"""CSLP multigrid V-cycle on the GPU (drop-in for reference mg.py:27-139).

Sub-hierarchy, smoother and transfers follow the reference: 5-point
rediscretised shifted operators on grids coarsened by k^2 injection while
both interval counts are even, min(nx, ny) > 5 and depth < mg_levels;
V(pre, post) damped Jacobi (omega 0.8); residual -> (1,4,6,4,1)/16
restriction with coarse Dirichlet rows zeroed -> recursion from zero ->
prolong-add -> post-smoothing; coarsest level solved directly when it has at
most ``direct_coarsest_limit`` points (dense inverse applied as a device GEMV;
the reference uses scipy LU) else by GMRES(coarsest_rule); divergence guard
||b - M x|| > guard * max(r0, ||b||) raises MgDivergence.

The whole cycle is one host call into the library (csrc/engine.cu,
Multigrid::cycle) with no host synchronisation inside; the divergence guard
is evaluated on the device and raised at the next synchronisation point.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import device as dev
from ._lib import check, lib
from .errors import CapacityError
from .grid import DIRICHLET
from .krylov import StopRule
from .operators import LevelOperator, radius1_operator

__all__ = ["MgConfig", "CslpMultigrid", "assemble_radius1_dense"]


@dataclass(frozen=True)
class MgConfig:
    pre_smooth: int = 1
    post_smooth: int = 1
    smoother_damping: float = 0.8
    mg_levels: int = 12
    coarsest_rule: StopRule = StopRule(1e-8, 50)
    direct_coarsest_limit: int = 4096
    divergence_guard: float = 10.0

    def __post_init__(self):
        if self.pre_smooth + self.post_smooth < 1:
            raise ValueError("at least one smoothing step is required")
        if self.mg_levels < 2:
            raise ValueError("mg_levels must be >= 2")


@dataclass
class _SubLevel:
    op: LevelOperator
    lu: object = None  # truthy when the coarsest level is solved directly


def assemble_radius1_dense(op: LevelOperator, max_points: int = 4096) -> np.ndarray:
    """Dense matrix of a radius-1 level operator, including the ghost closure
    folded onto boundary columns and Dirichlet identity rows."""
    n = op.npoints
    if n > max_points:
        raise CapacityError(f"{n} points exceed the dense assembly guard {max_points}")
    ny, nx = op.shape
    s = op.lap_coef[1, 1] / 4.0
    mc = op.mass_coef[1, 1]
    k = np.sqrt(op.ksq)
    A = np.zeros((n, n), dtype=np.complex128)
    idx = np.arange(n).reshape(ny, nx)
    A[idx, idx] = 4.0 * s + mc * op.ksq
    for dj, di in ((0, -1), (0, 1), (-1, 0), (1, 0)):
        jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        tj, ti = jj + dj, ii + di
        inside = (tj >= 0) & (tj < ny) & (ti >= 0) & (ti < nx)
        A[idx[inside], idx[tj[inside], ti[inside]]] += -s
    w, e, so, no = op.boundary
    two_ih = 2.0j * op.h
    # ghost taps (coefficient -s) folded onto (boundary, inner) columns
    for kind, rows, bcol, icol, kb in (
            (w, idx[:, 0], idx[:, 0], idx[:, 1], k[:, 0]),
            (e, idx[:, -1], idx[:, -1], idx[:, -2], k[:, -1]),
            (so, idx[0, :], idx[0, :], idx[1, :], k[0, :]),
            (no, idx[-1, :], idx[-1, :], idx[-2, :], k[-1, :])):
        if kind == DIRICHLET:
            A[rows, bcol] += -s * 2.0
            A[rows, icol] += -s * -1.0
        else:
            A[rows, bcol] += -s * two_ih * kb
            A[rows, icol] += -s
    for sl in op.dirichlet_slices():
        r = idx[sl]
        A[r, :] = 0.0
        A[r, r] = 1.0
    return A


class CslpMultigrid:
    """V-cycle for ``-Laplace - (beta1 + i beta2) I(k^2)`` on one grid (GPU)."""

    def __init__(self, nx, ny, h, ksq, boundary, beta2, beta1=1.0, config: MgConfig = MgConfig(),
                 slabs=None):
        """slabs: optional callable sub-level index -> distributed.SlabSpec or None
        (row-slab decomposition of the sub-hierarchy; None everywhere = one rank)."""
        self.config = config
        shift = complex(beta1, beta2)
        self.levels: list[_SubLevel] = []
        cx, cy, ch = int(nx), int(ny), float(h)
        on_device = dev.is_device(ksq)  # GPU-built hierarchy: sub-level k^2 by injection on the device
        kk = dev.to_device(ksq, dtype="f8") if on_device else np.ascontiguousarray(ksq, dtype=np.float64)
        while True:
            sl = slabs(len(self.levels)) if slabs is not None else None
            self.levels.append(_SubLevel(op=radius1_operator(cx, cy, ch, kk, boundary, shift, slab=sl)))
            if not ((cx - 1) % 2 == 0 and (cy - 1) % 2 == 0 and min(cx, cy) > 5
                    and len(self.levels) < config.mg_levels):
                break
            cx, cy, ch = (cx - 1) // 2 + 1, (cy - 1) // 2 + 1, 2.0 * ch
            if on_device:
                nxt = dev.empty((cy, cx), dtype="f8")
                check(lib().hdb_setup_inject(kk.data_ptr(), kk.shape[1], kk.shape[0], nxt.data_ptr()))
                kk = nxt
            else:
                kk = kk[::2, ::2].copy()
        last = self.levels[-1]
        self._inv = None
        if last.op.npoints <= config.direct_coarsest_limit:
            self._inv = np.ascontiguousarray(np.linalg.inv(assemble_radius1_dense(last.op)))
            last.lu = True
        self._handle = None

    @property
    def depth(self) -> int:
        return len(self.levels)

    @property
    def handle(self):
        if self._handle is None:
            ops = (C.c_void_p * self.depth)(*[lv.op.handle.value for lv in self.levels])
            inv = self._inv.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)) if self._inv is not None else None
            ninv = self._inv.shape[0] if self._inv is not None else 0
            cfg = self.config
            h = C.c_void_p()
            check(lib().hdb_mg_create(C.byref(h), ops, self.depth, inv, ninv, float(cfg.smoother_damping),
                                      int(cfg.pre_smooth), int(cfg.post_smooth), float(cfg.divergence_guard),
                                      float(cfg.coarsest_rule.rel_tol), int(cfg.coarsest_rule.max_iters)))
            self._handle = h
        return self._handle

    def close(self):
        if self._handle is not None:
            from . import _lib
            if _lib._lib is not None:
                _lib._lib.hdb_mg_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _device_apply(self, pin, pout):
        check(lib().hdb_mg_vcycle(self.handle, pin, None, pout))

    def vcycle(self, b, x0=None):
        """One V-cycle toward the solution of the shifted system (mg.py:125-139)."""
        host = not dev.is_device(b)
        db = dev.to_device(b)
        dx0 = dev.to_device(x0) if x0 is not None else None
        out = dev.empty(tuple(b.shape))
        check(lib().hdb_mg_vcycle(self.handle, db.data_ptr(), dx0.data_ptr() if dx0 is not None else None,
                                  out.data_ptr()))
        return dev.to_host(out) if host else out
