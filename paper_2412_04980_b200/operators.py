"""Matrix-free level operators on the GPU (drop-in for reference operators.py).

``LevelOperator`` keeps the reference constructor, attributes and methods
(operators.py:96-208): coefficients are converted to float exactly once, the
same way (lap_coef = num/den/h^2, mass_coef = (-shift/level_scale)*num/den),
and handed to the CUDA library; ``apply`` runs the sm_100a kernel
(csrc/kernels_stencil.cu), bit-identical to the reference's numba loop.

Inputs may be numpy arrays (copied to the device and back, the reference's
calling convention) or torch CUDA complex128 tensors (no copies).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import device as dev
from ._lib import check, lib
from .errors import ShapeError
from .grid import BC_CODE, DIRICHLET, ComplexField
from .stencils import StencilKernel, level_kernels, mass_level_scale

__all__ = ["LevelOperator", "helmholtz_operator", "cslp_operator", "radius1_operator",
           "apply_helmholtz", "apply_cslp", "matvec_flop_byte_counters", "arithmetic_intensity",
           "ALGORITHMIC_BYTES_PER_POINT"]

# algorithmic HBM bytes per grid point: u 16 + k^2 8 + out 16
ALGORITHMIC_BYTES_PER_POINT = {"apply": 40, "residual": 56, "jacobi": 56, "jacobi0": 40}


class LevelOperator:
    """Matrix-free ``-Laplace - shift * I(k^2)`` on one grid level (GPU)."""

    def __init__(self, level, nx, ny, h, ksq, boundary, laplace: StencilKernel, mass: StencilKernel,
                 shift=1.0, level_scale=1.0, slab=None):
        if laplace.radius != mass.radius:
            raise ShapeError("laplace and mass kernels must share a radius")
        self.level = level
        self.nx, self.ny, self.h = int(nx), int(ny), float(h)
        self.ksq = np.ascontiguousarray(ksq, dtype=np.float64)
        if self.ksq.shape != (self.ny, self.nx):
            raise ShapeError(f"k^2 shape {self.ksq.shape} != {(self.ny, self.nx)}")
        self.boundary = tuple(boundary)
        self.shift = complex(shift)
        self.radius = laplace.radius
        self.laplace, self.mass = laplace, mass
        # float conversion, once (operators.py:111-113)
        self.lap_coef = laplace.as_float() / self.h ** 2
        self.mass_coef = (-self.shift / level_scale) * mass.as_float().astype(np.complex128)
        self.slab = slab  # distributed.SlabSpec of this rank, None = whole grid
        self._handle = None

    # -- device handle ------------------------------------------------------
    @property
    def handle(self):
        if self._handle is None:
            L = lib()
            h = C.c_void_p()
            bc = (C.c_int * 4)(*[BC_CODE[b] for b in self.boundary])
            lap = np.ascontiguousarray(self.lap_coef, dtype=np.float64)
            mre = np.ascontiguousarray(self.mass_coef.real)
            mim = np.ascontiguousarray(self.mass_coef.imag)
            f = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
            if self.slab is None:
                check(L.hdb_op_create(C.byref(h), self.nx, self.ny, self.radius, self.h, bc, f(lap), f(mre), f(mim),
                                      f(self.ksq)))
            else:
                sl = self.slab
                P = len(sl.table_row0)
                r0s = (C.c_int * P)(*sl.table_row0)
                nys = (C.c_int * P)(*sl.table_ny)
                check(L.hdb_op_create_slab(C.byref(h), self.nx, self.ny, self.radius, self.h, bc, f(lap), f(mre),
                                           f(mim), f(self.ksq), sl.row0, sl.ny, sl.halo, P, r0s, nys))
            self._handle = h
        return self._handle

    def close(self):
        if self._handle is not None:
            from . import _lib
            if _lib._lib is not None:
                _lib._lib.hdb_op_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def shape(self):
        return (self.ny, self.nx)

    @property
    def npoints(self):
        return self.nx * self.ny

    def dirichlet_slices(self):
        w, e, s, n = self.boundary
        out = []
        if w == DIRICHLET:
            out.append((slice(None), 0))
        if e == DIRICHLET:
            out.append((slice(None), -1))
        if s == DIRICHLET:
            out.append((0, slice(None)))
        if n == DIRICHLET:
            out.append((-1, slice(None)))
        return out

    def dirichlet_mask(self) -> int:
        return sum(1 << i for i, b in enumerate(self.boundary) if b == DIRICHLET)

    # -- compute --------------------------------------------------------------
    def _io(self, u, *more):
        if tuple(u.shape) != self.shape:
            raise ShapeError(f"field shape {tuple(u.shape)} does not match level grid {self.shape}")
        host = not dev.is_device(u)
        ts = [dev.to_device(a) for a in (u,) + more]
        return host, ts

    def apply(self, u, out=None, pool=None, tiles=None):
        """v = A u (operators.py:130-147); pool/tiles accepted for API compatibility."""
        host, (du,) = self._io(u)
        dout = dev.empty(self.shape) if (out is None or not dev.is_device(out)) else out
        check(lib().hdb_op_apply(self.handle, du.data_ptr(), dout.data_ptr()))
        if host:
            res = dev.to_host(dout)
            if out is not None:
                out[...] = res
                return out
            return res
        return dout

    def _device_apply(self, pin, pout):
        check(lib().hdb_op_apply(self.handle, pin, pout))

    def residual(self, b, u):
        """r = b - A u (fused; Dirichlet rows give b - u)."""
        host, (du, db) = self._io(u, b)
        dout = dev.empty(self.shape)
        check(lib().hdb_op_residual(self.handle, db.data_ptr(), du.data_ptr(), dout.data_ptr()))
        return dev.to_host(dout) if host else dout

    def residual_norms(self, b, u):
        """(||b - A u||, ||b||) from one fused pass (the MG divergence guard's
        quantities, mg.py:131-138); the residual is not stored."""
        _, (du, db) = self._io(u, b)
        out = (C.c_double * 2)()
        check(lib().hdb_op_resnorm(self.handle, db.data_ptr(), du.data_ptr(), out))
        return float(np.sqrt(max(out[0], 0.0))), float(np.sqrt(max(out[1], 0.0)))

    def jacobi(self, x, b, omega=0.8):
        """One damped Jacobi sweep out of place (mg.py:88-102); x=None: from zero."""
        if x is None:
            host, (db,) = self._io(b)
            xp = None
        else:
            host, (dx, db) = self._io(x, b)
            xp = dx.data_ptr()
        dout = dev.empty(self.shape)
        check(lib().hdb_op_jacobi(self.handle, xp, db.data_ptr(), dout.data_ptr(), float(omega)))
        return dev.to_host(dout) if host else dout

    def diagonal(self) -> np.ndarray:
        """Matrix diagonal incl. ghost-closure terms (operators.py:180-208), host setup."""
        if self.radius != 1:
            raise ShapeError("diagonal is only provided for radius-1 operators")
        s = self.lap_coef[1, 1] / 4.0
        d = np.full(self.shape, 4.0 * s, dtype=np.complex128)
        d += self.mass_coef[1, 1] * self.ksq
        k = np.sqrt(self.ksq)
        sides = ((slice(None), 0), (slice(None), -1), (0, slice(None)), (-1, slice(None)))
        edges = (k[:, 0], k[:, -1], k[0, :], k[-1, :])
        for kind, sl, ke in zip(self.boundary, sides, edges):
            if kind != DIRICHLET:
                d[sl] += -s * 2.0j * self.h * ke
        for kind, sl in zip(self.boundary, sides):
            if kind == DIRICHLET:
                d[sl] = 1.0
        return d

    def assemble_dense(self) -> np.ndarray:
        """Explicit matrix by probing the GPU operator with unit vectors (small grids).

        Column c is A e_c; the probes are batched through one device buffer."""
        n = self.npoints
        if n > 40_000:
            from .errors import CapacityError
            raise CapacityError(f"{n} points exceed the dense assembly guard")
        torch = dev.torch_mod()
        A = np.empty((n, n), dtype=np.complex128)
        e = torch.zeros(self.shape, dtype=torch.complex128, device="cuda")
        out = torch.empty_like(e)
        flat = e.view(-1)
        for c in range(n):
            flat[c] = 1.0
            check(lib().hdb_op_apply(self.handle, e.data_ptr(), out.data_ptr()))
            A[:, c] = out.view(-1).cpu().numpy()
            flat[c] = 0.0
        return A


def _level_operator(hierarchy, level, shift, slab=None):
    lv = hierarchy.level(level)
    lap, mass = level_kernels(level)
    return LevelOperator(level, lv.nx, lv.ny, lv.h, hierarchy.ksq_at(level), hierarchy.boundary, lap, mass,
                         shift=shift, level_scale=mass_level_scale(level), slab=slab)


def helmholtz_operator(hierarchy, level: int, slab=None) -> LevelOperator:
    return _level_operator(hierarchy, level, 1.0, slab)


def cslp_operator(hierarchy, level: int, beta2: float, beta1: float = 1.0, slab=None) -> LevelOperator:
    return _level_operator(hierarchy, level, complex(beta1, beta2), slab)


def radius1_operator(nx, ny, h, ksq, boundary, shift, slab=None) -> LevelOperator:
    lap, mass = level_kernels(1)
    return LevelOperator(0, nx, ny, h, ksq, boundary, lap, mass, shift=shift, level_scale=1.0, slab=slab)


def apply_helmholtz(op: LevelOperator, hierarchy, u: ComplexField) -> ComplexField:
    if u.level != op.level:
        raise ShapeError(f"field level {u.level} does not match operator level {op.level}")
    return ComplexField(level=u.level, data=np.asarray(op.apply(u.grid_view(hierarchy))).ravel())


def apply_cslp(op: LevelOperator, hierarchy, u: ComplexField) -> ComplexField:
    return apply_helmholtz(op, hierarchy, u)


def matvec_flop_byte_counters(kind: str, n_points: int):
    """Reference roofline model (operators.py:337-352): 11 flop/56 B MF, 10/120 CSR."""
    if kind == "matrix_free":
        return 11 * n_points, 56 * n_points
    if kind == "csr":
        return 10 * n_points, 120 * n_points
    raise ValueError(f"unknown matvec kind {kind!r}")


def arithmetic_intensity(kind: str) -> float:
    f, b = matvec_flop_byte_counters(kind, 1)
    return f / b
