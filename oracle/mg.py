"""CSLP multigrid V(1,1) (oracle restatement of mg.py:51-139).

Sub-hierarchy by k^2 injection while both interval counts are even, more than
5 points per direction and fewer than mg_levels levels (mg.py:65-79); damped
Jacobi omega=0.8; residual -> [1,4,6,4,1] restriction with coarse Dirichlet
rows zeroed -> recurse from zero -> prolong-add -> post-smooth (mg.py:111-123);
coarsest dense LU (<= 4096 points) else GMRES(1e-8, 50) with np.vdot
(mg.py:81-82,104-109); divergence guard 10x (mg.py:125-139).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .krylov import Stop, fgmres
from .ops import prolong, radius1_op, restrict


class MgDivergenceOracle(RuntimeError):
    pass


def dense_matrix(op):
    """Explicit matrix of a level operator, entry order of assemble_csr
    (operators.py:261-328): per row, offsets row-major, ghost taps folded onto
    (boundary, inner) columns with weights (2, -1) Dirichlet or (2ih k_b, 1)
    Sommerfeld, duplicates summed by scipy's COO->CSR conversion."""
    import scipy.sparse as sp
    from .grid import DIRICHLET
    nx, ny, r = op.nx, op.ny, op.r
    w_, e_, s_, n_ = op.boundary
    kw, ke, ks, kn = op.kedge
    rows, cols, vals = [], [], []

    def ghost(kind, kb):
        return (2.0 + 0.0j, -1.0 + 0.0j) if kind == DIRICHLET else (2.0j * op.h * kb, 1.0 + 0.0j)

    for j in range(ny):
        for i in range(nx):
            row = j * nx + i
            if ((w_ == DIRICHLET and i == 0) or (e_ == DIRICHLET and i == nx - 1)
                    or (s_ == DIRICHLET and j == 0) or (n_ == DIRICHLET and j == ny - 1)):
                rows.append(row); cols.append(row); vals.append(1.0 + 0.0j)  # noqa: E702
                continue
            for oj in range(-r, r + 1):
                for oi in range(-r, r + 1):
                    ii, jj = i + oi, j + oj
                    coef = op.lap[oj + r, oi + r] + op.mass[oj + r, oi + r] * op.kpad[jj + r, ii + r]
                    if coef == 0:
                        continue
                    xin, yin = 0 <= ii < nx, 0 <= jj < ny
                    taps = None
                    if xin and yin:
                        taps = ((jj * nx + ii, coef),)
                    elif yin and ii == -1:
                        wb, wi = ghost(w_, kw[jj]); taps = ((jj * nx, coef * wb), (jj * nx + 1, coef * wi))  # noqa: E702
                    elif yin and ii == nx:
                        wb, wi = ghost(e_, ke[jj]); taps = ((jj * nx + nx - 1, coef * wb), (jj * nx + nx - 2, coef * wi))  # noqa: E702,E501
                    elif xin and jj == -1:
                        wb, wi = ghost(s_, ks[ii]); taps = ((ii, coef * wb), (nx + ii, coef * wi))  # noqa: E702
                    elif xin and jj == ny:
                        wb, wi = ghost(n_, kn[ii]); taps = (((ny - 1) * nx + ii, coef * wb), ((ny - 2) * nx + ii, coef * wi))  # noqa: E702,E501
                    for c, v in taps or ():
                        rows.append(row); cols.append(c); vals.append(v)  # noqa: E702
    n = nx * ny
    m = sp.coo_matrix((np.array(vals, dtype=np.complex128), (rows, cols)), shape=(n, n))
    return m.tocsr().toarray()


class CpuMultigrid:
    def __init__(self, nx, ny, h, ksq, boundary, beta2, beta1=1.0, pre=1, post=1, omega=0.8,
                 mg_levels=12, direct_limit=4096, guard=10.0, coarse_stop=Stop(1e-8, 50)):
        shift = complex(beta1, beta2)
        self.pre, self.post, self.omega, self.guard = pre, post, omega, guard
        self.coarse_stop = coarse_stop
        self.ops = []
        cx, cy, ch, kk = nx, ny, float(h), np.ascontiguousarray(ksq, dtype=np.float64)
        while True:
            op = radius1_op(cx, cy, ch, kk, boundary, shift)
            op.diagonal()
            self.ops.append(op)
            if not ((cx - 1) % 2 == 0 and (cy - 1) % 2 == 0 and min(cx, cy) > 5
                    and len(self.ops) < mg_levels):
                break
            cx, cy, ch, kk = (cx - 1) // 2 + 1, (cy - 1) // 2 + 1, 2.0 * ch, kk[::2, ::2].copy()
        last = self.ops[-1]
        self.lu = sla.lu_factor(dense_matrix(last)) if last.nx * last.ny <= direct_limit else None

    @property
    def depth(self):
        return len(self.ops)

    def _coarse(self, b):
        op = self.ops[-1]
        if self.lu is not None:
            return sla.lu_solve(self.lu, b.ravel()).reshape(b.shape)
        x, _ = fgmres(op.apply, None, b, self.coarse_stop)
        return x

    def _cycle(self, i, b, x):
        if i == len(self.ops) - 1:
            return self._coarse(b)
        op = self.ops[i]
        x = op.jacobi(x, b, self.omega, self.pre)
        r = b - op.apply(x)
        rc = restrict(r)
        for sl in self.ops[i + 1].pinned():
            rc[sl] = 0.0
        ec = self._cycle(i + 1, rc, np.zeros_like(rc))
        x = x + prolong(ec, b.shape)
        return op.jacobi(x, b, self.omega, self.post)

    def vcycle(self, b):
        x = np.zeros_like(b)
        bn = np.linalg.norm(b)
        if bn == 0.0:
            return x
        x = self._cycle(0, b, x)
        post = np.linalg.norm(b - self.ops[0].apply(x))
        if post > self.guard * bn:
            raise MgDivergenceOracle(f"V-cycle residual grew from {bn:.3e} to {post:.3e}")
        return x
