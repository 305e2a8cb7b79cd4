"""Matrix-free level operators, Jacobi, transfers and dots (oracle restatement).

Arithmetic follows the reference operation-for-operation so results are
bit-identical to it on the same host:
  * ghost closure            operators.py:44-93
  * coefficient conversion   operators.py:99-117
  * radius-1 / general loops _kernels.py:14-50 (numba, no fastmath => no FMA)
  * Dirichlet identity rows  operators.py:163-166
  * Jacobi diagonal          operators.py:180-208, sweep _kernels.py:53-68
  * transfers                transfers.py:59-88 (strided numpy passes)
  * reduce_dot               parallel.py:168-195 (64-row blocks, np.vdot)
"""
from __future__ import annotations

import numba as nb
import numpy as np

from .chain import level_kernels, mass_level_scale
from .grid import DIRICHLET

_njit = nb.njit(cache=False, nogil=True)

# Row-slab worker pool for the stencil loops (the reference runs its numba
# kernels on disjoint output tiles in a ThreadPoolExecutor, parallel.py:1-7 and
# WorkerPool).  Each slab computes the same per-point arithmetic, so results are
# bit-identical for any worker count; 1 worker (the default, and what the tests
# use) runs the loops inline.
_WORKERS = 1
_POOL = None


def set_workers(n: int) -> int:
    """Use up to `n` host threads for the stencil loops; returns the count set."""
    global _WORKERS, _POOL
    n = max(1, int(n))
    if n != _WORKERS:
        if _POOL is not None:
            _POOL.shutdown()
            _POOL = None
        _WORKERS = n
        if n > 1:
            from concurrent.futures import ThreadPoolExecutor
            _POOL = ThreadPoolExecutor(max_workers=n)
    return _WORKERS


def workers() -> int:
    return _WORKERS


def _row_slabs(fn, ny, halo, padded_args, plain_args, scalars, out):
    """fn(*padded[j0:j1+2*halo], *plain[j0:j1], out[j0:j1], *scalars) over row slabs."""
    if _WORKERS == 1 or ny < 64:
        fn(*padded_args, *plain_args, out, *scalars)
        return
    parts = min(_WORKERS, ny // 32)
    cuts = [ny * t // parts for t in range(parts + 1)]
    futs = [_POOL.submit(fn, *[a[j0:j1 + 2 * halo] for a in padded_args], *[a[j0:j1] for a in plain_args],
                         out[j0:j1], *scalars) for j0, j1 in zip(cuts[:-1], cuts[1:])]
    for f in futs:
        f.result()


@_njit
def _five_point(up, ksq, out, s, mc):
    ny, nx = out.shape
    for j in range(ny):
        for i in range(nx):
            c = up[j + 1, i + 1]
            lap = 4.0 * c - up[j + 1, i] - up[j + 1, i + 2] - up[j, i + 1] - up[j + 2, i + 1]
            out[j, i] = s * lap + mc * ksq[j, i] * c


@_njit
def _dense_taps(up, kp, out, lap, mass):
    ny, nx = out.shape
    n = lap.shape[0]
    for j in range(ny):
        for i in range(nx):
            acc = 0.0 + 0.0j
            for a in range(n):
                for b in range(n):
                    acc += (lap[a, b] + mass[a, b] * kp[j + a, i + b]) * up[j + a, i + b]
            out[j, i] = acc


@_njit
def _jacobi_sweep(up, ksq, rhs, dinv, out, s, mc, omega):
    ny, nx = out.shape
    for j in range(ny):
        for i in range(nx):
            c = up[j + 1, i + 1]
            lap = 4.0 * c - up[j + 1, i] - up[j + 1, i + 2] - up[j, i + 1] - up[j + 2, i + 1]
            mu = s * lap + mc * ksq[j, i] * c
            out[j, i] = c + omega * dinv[j, i] * (rhs[j, i] - mu)


class CpuLevelOp:
    """-Laplace - shift*I(k^2) on one level (operators.py:96-208)."""

    def __init__(self, nx, ny, h, ksq, boundary, lap_tab, lap_den, mass_tab, mass_den,
                 shift=1.0, level_scale=1.0):
        self.nx, self.ny, self.h = nx, ny, float(h)
        self.ksq = np.ascontiguousarray(ksq, dtype=np.float64)
        self.boundary = tuple(boundary)
        self.shift = complex(shift)
        self.r = len(lap_tab) // 2
        self.lap = np.array(lap_tab, dtype=np.float64) / float(lap_den) / self.h ** 2
        self.mass = (-self.shift / level_scale) * (
            np.array(mass_tab, dtype=np.float64) / float(mass_den)).astype(np.complex128)
        kf = np.sqrt(self.ksq)
        self.kedge = (kf[:, 0], kf[:, -1], kf[0, :], kf[-1, :])
        self.kpad = self._pad_ksq()
        self._dinv = None

    @property
    def shape(self):
        return (self.ny, self.nx)

    # ghost closure ---------------------------------------------------------
    def pad(self, u):
        r, ny, nx = self.r, self.ny, self.nx
        p = np.zeros((ny + 2 * r, nx + 2 * r), dtype=np.complex128)
        p[r:r + ny, r:r + nx] = u
        w_, e_, s_, n_ = self.boundary
        kw, ke, ks, kn = self.kedge
        tih = 2.0j * self.h
        p[r:r + ny, r - 1] = 2.0 * u[:, 0] - u[:, 1] if w_ == DIRICHLET else u[:, 1] + tih * kw * u[:, 0]
        p[r:r + ny, r + nx] = 2.0 * u[:, -1] - u[:, -2] if e_ == DIRICHLET else u[:, -2] + tih * ke * u[:, -1]
        p[r - 1, r:r + nx] = 2.0 * u[0, :] - u[1, :] if s_ == DIRICHLET else u[1, :] + tih * ks * u[0, :]
        p[r + ny, r:r + nx] = 2.0 * u[-1, :] - u[-2, :] if n_ == DIRICHLET else u[-2, :] + tih * kn * u[-1, :]
        return p

    def _pad_ksq(self):
        r, ny, nx, k = self.r, self.ny, self.nx, self.ksq
        p = np.zeros((ny + 2 * r, nx + 2 * r))
        p[r:r + ny, r:r + nx] = k
        w_, e_, s_, n_ = self.boundary
        if w_ == DIRICHLET:
            p[r:r + ny, r - 1] = 2.0 * k[:, 0] - k[:, 1]
        if e_ == DIRICHLET:
            p[r:r + ny, r + nx] = 2.0 * k[:, -1] - k[:, -2]
        if s_ == DIRICHLET:
            p[r - 1, r:r + nx] = 2.0 * k[0, :] - k[1, :]
        if n_ == DIRICHLET:
            p[r + ny, r:r + nx] = 2.0 * k[-1, :] - k[-2, :]
        return p

    def pinned(self):
        w_, e_, s_, n_ = self.boundary
        sl = []
        if w_ == DIRICHLET:
            sl.append((slice(None), 0))
        if e_ == DIRICHLET:
            sl.append((slice(None), -1))
        if s_ == DIRICHLET:
            sl.append((0, slice(None)))
        if n_ == DIRICHLET:
            sl.append((-1, slice(None)))
        return sl

    # application -------------------------------------------------------------
    def apply(self, u):
        u = np.asarray(u, dtype=np.complex128)
        if u.shape != self.shape:
            raise ValueError(f"shape {u.shape} != {self.shape}")
        up = self.pad(u)
        out = np.empty_like(u)
        if self.r == 1:
            _row_slabs(_five_point, self.ny, 1, (up,), (self.ksq,), (self.lap[1, 1] / 4.0, self.mass[1, 1]), out)
        else:
            _row_slabs(lambda up_, kp_, o_: _dense_taps(up_, kp_, o_, self.lap, self.mass), self.ny, self.r,
                       (up, self.kpad), (), (), out)
        for sl in self.pinned():
            out[sl] = u[sl]
        return out

    def diagonal(self):
        """operators.py:180-208 (radius 1 only)."""
        if self._dinv is not None:
            return self._diag
        s = self.lap[1, 1] / 4.0
        d = np.full(self.shape, 4.0 * s, dtype=np.complex128)
        d += self.mass[1, 1] * self.ksq
        sides = ((slice(None), 0), (slice(None), -1), (0, slice(None)), (-1, slice(None)))
        for kind, sl, ke in zip(self.boundary, sides, self.kedge):
            if kind != DIRICHLET:
                d[sl] += -s * 2.0j * self.h * ke
        for kind, sl in zip(self.boundary, sides):
            if kind == DIRICHLET:
                d[sl] = 1.0
        self._diag = d
        self._dinv = 1.0 / d
        return d

    def dinv(self):
        self.diagonal()
        return self._dinv

    def jacobi(self, x, b, omega, sweeps=1):
        """mg.py:88-102: damped Jacobi, Dirichlet rows relax toward data."""
        dinv = self.dinv()
        for _ in range(sweeps):
            out = np.empty_like(x)
            _row_slabs(_jacobi_sweep, self.ny, 1, (self.pad(x),), (self.ksq, b, dinv),
                       (self.lap[1, 1] / 4.0, self.mass[1, 1], omega), out)
            for sl in self.pinned():
                out[sl] = x[sl] + omega * (b[sl] - x[sl])
            x = out
        return x


def radius1_op(nx, ny, h, ksq, boundary, shift):
    """operators.py:235-238 (MG sub-levels: 5-point pair, level_scale 1)."""
    lt, ld, mt, md, _ = level_kernels(1)
    return CpuLevelOp(nx, ny, h, ksq, boundary, lt, ld, mt, md, shift=shift, level_scale=1.0)


def _level_op(hier, l, shift):
    lv = hier.level(l)
    lt, ld, mt, md, _ = level_kernels(l)
    return CpuLevelOp(lv.nx, lv.ny, lv.h, hier.ksq_at(l), hier.boundary, lt, ld, mt, md,
                      shift=shift, level_scale=mass_level_scale(l))


def helmholtz_op(hier, l):
    """operators.py:215-222 (shift 1)."""
    return _level_op(hier, l, 1.0)


def cslp_op(hier, l, beta2, beta1=1.0):
    """operators.py:225-232 (shift beta1 + i beta2)."""
    return _level_op(hier, l, complex(beta1, beta2))


# transfers -------------------------------------------------------------------
_W16 = np.array([1, 4, 6, 4, 1], dtype=np.float64) / 16   # transfers.py:49
_W8 = np.array([1, 4, 6, 4, 1], dtype=np.float64) / 8     # transfers.py:50


def restrict(fine):
    """transfers.py:59-72: 25 strided passes in (b, a) row-major order."""
    ny, nx = fine.shape
    if (nx - 1) % 2 or (ny - 1) % 2:
        raise ValueError("cannot coarsen")
    ncy, ncx = (ny - 1) // 2 + 1, (nx - 1) // 2 + 1
    pad = np.zeros((ny + 4, nx + 4), dtype=fine.dtype)
    pad[2:-2, 2:-2] = fine
    out = np.zeros((ncy, ncx), dtype=fine.dtype)
    for b in range(5):
        for a in range(5):
            out += (_W16[b] * _W16[a]) * pad[b:b + 2 * ncy - 1:2, a:a + 2 * ncx - 1:2]
    return out


def prolong(coarse, fine_shape):
    """transfers.py:75-88: scatter-accumulate in (b, a) row-major order."""
    nfy, nfx = fine_shape
    ncy, ncx = coarse.shape
    if nfx != 2 * ncx - 1 or nfy != 2 * ncy - 1:
        raise ValueError("shape mismatch")
    pad = np.zeros((nfy + 4, nfx + 4), dtype=coarse.dtype)
    for b in range(5):
        for a in range(5):
            pad[b:b + 2 * ncy - 1:2, a:a + 2 * ncx - 1:2] += (_W8[b] * _W8[a]) * coarse
    return pad[2:-2, 2:-2]


# dots ------------------------------------------------------------------------
_ROWS = 64  # parallel.py:30


def reduce_dot(u, v):
    """parallel.py:168-195: conj(u).v over fixed 64-row blocks, ascending."""
    u2 = u.reshape(1, -1) if u.ndim == 1 else u
    v2 = v.reshape(1, -1) if v.ndim == 1 else v
    ny = u2.shape[0]
    nb_ = -(ny // -_ROWS)
    if nb_ == 1:
        return complex(np.vdot(u2, v2))
    part = np.empty(nb_, dtype=np.complex128)
    for t in range(nb_):
        part[t] = np.vdot(u2[t * _ROWS:(t + 1) * _ROWS], v2[t * _ROWS:(t + 1) * _ROWS])
    return complex(np.add.reduce(part))
