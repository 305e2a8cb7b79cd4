"""MADP preset and A-DEF1 recursive solver (oracle restatement of madp.py).

preset("MADP")  madp.py:129-189 (beta2 = 0.5; CSLP = MG on levels 1-2 unless
coarsest, GMRES(0.1, ceil(6 N^1/4)) elsewhere; level-2 cycle (0.3, 100);
levels 3..ml-1 (1, 1); coarsest (0.1, 100) if indefinite else (1, 1);
NegDef iff max k*h_l >= 2, monotone, madp.py:77-84).
Recursion  madp.py:301-327, outer solve madp.py:329-371, CSLP dispatch
madp.py:277-299.  Also restates MADP_V1/V2/V3 policies for completeness.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .krylov import Stop, cslp_cap, fgmres
from .mg import CpuMultigrid
from .ops import cslp_op, helmholtz_op, prolong, reduce_dot, restrict


@dataclass(frozen=True)
class Pol:
    level: int
    cslp: str          # "mg" | "gmres" | "none"
    beta2: float
    cslp_stop: Stop
    cycle: Stop | None


def madp_preset(hier, name="MADP", outer=Stop(1e-6, 150), threshold=2.0):
    ml = hier.ml
    neg, flipped = [], False
    for l in range(1, ml + 1):
        flipped = flipped or float(np.sqrt(hier.ksq_at(l).max()) * hier.level(l).h) >= threshold
        neg.append(flipped)
    lx, ly = hier.extent
    kdim = float(np.sqrt(hier.ksq_at(1).max() * lx * ly))
    if name in ("MADP_V1", "MADP_V2"):
        beta = {l: 1.0 / kdim for l in range(1, ml + 1)}
        meth = {l: "gmres" for l in range(1, ml + 1)}
        l2 = Stop(0.1, 100) if name == "MADP_V2" else Stop(1.0, 1)
    else:
        beta = {l: 0.5 for l in range(1, ml + 1)}
        meth = {l: ("mg" if l <= 2 else "gmres") for l in range(1, ml + 1)}
        meth[ml] = "gmres"
        l2 = Stop(0.3 if name == "MADP" else 0.1, 100)
    coarsest = Stop(1.0, 1) if neg[-1] else Stop(0.1, 100)
    pols = []
    for l in range(1, ml + 1):
        cyc = None if l == 1 else coarsest if l == ml else l2 if l == 2 else Stop(1.0, 1)
        pols.append(Pol(l, meth[l], beta[l], Stop(0.1, cslp_cap(hier.level(l).npoints)), cyc))
    return pols, outer


class CpuMadpSolver:
    def __init__(self, hier, policies, outer):
        self.h, self.pols, self.outer = hier, policies, outer
        self.A, self.M, self.mg = {}, {}, {}
        for l in range(1, hier.ml + 1):
            p = policies[l - 1]
            self.A[l] = helmholtz_op(hier, l)
            if p.cslp == "gmres":
                self.M[l] = cslp_op(hier, l, p.beta2)
            elif p.cslp == "mg":
                lv = hier.level(l)
                self.mg[l] = CpuMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(l), hier.boundary, p.beta2)

    def _reset(self):
        ml = self.h.ml
        self.cycle_iters = {l: [] for l in range(2, ml + 1)}
        self.cslp_iters = {l: [] for l in range(1, ml + 1)}
        self.matvecs = {l: 0 for l in range(1, ml + 1)}

    def _Aop(self, l):
        def f(u):
            self.matvecs[l] += 1
            return self.A[l].apply(u)
        return f

    def _cslp(self, l, rhs):
        p = self.pols[l - 1]
        if p.cslp == "none":
            return rhs.copy()
        if p.cslp == "mg":
            self.cslp_iters[l].append(1)
            return self.mg[l].vcycle(rhs)
        x, rep = fgmres(self.M[l].apply, None, rhs, p.cslp_stop, dot=reduce_dot)
        self.cslp_iters[l].append(rep.iterations)
        return x

    def precond(self, l, v):
        nxt = l + 1
        vhat = restrict(v)
        stop = self.pols[nxt - 1].cycle
        if nxt == self.h.ml:
            inner = lambda w: self._cslp(nxt, w)  # noqa: E731
        else:
            inner = lambda w: self.precond(nxt, w)  # noqa: E731
        vtil, rep = fgmres(self._Aop(nxt), inner, vhat, stop, dot=reduce_dot)
        self.cycle_iters[nxt].append(rep.iterations)
        t = prolong(vtil, v.shape)
        s = self._Aop(l)(t)
        r = self._cslp(l, v - s)
        return r + t

    def solve(self, b, max_outer=None):
        self._reset()
        stop = self.outer if max_outer is None else Stop(self.outer.rel_tol, max_outer)
        t0 = time.perf_counter()
        x, rep = fgmres(self._Aop(1), lambda v: self.precond(1, v), b, stop, dot=reduce_dot)
        rep.wall_s = time.perf_counter() - t0
        return x, rep
