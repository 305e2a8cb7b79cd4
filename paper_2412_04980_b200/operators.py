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

__all__ = ["LevelOperator", "helmholtz_operator", "cslp_operator", "radius1_operator", "ghost_pad",
           "ksq_ghost_pad", "apply_helmholtz", "apply_cslp", "assemble_csr", "assemble_dense",
           "matvec_flop_byte_counters", "arithmetic_intensity", "ALGORITHMIC_BYTES_PER_POINT"]

DEFAULT_ASSEMBLY_LIMIT = 1_100_000  # points (operators.py:41)

# algorithmic HBM bytes per grid point: u 16 + k^2 8 + out 16
ALGORITHMIC_BYTES_PER_POINT = {"apply": 40, "residual": 56, "jacobi": 56, "jacobi0": 40}


# ghost column/row of each side (west, east, south, north): where it lies in the
# padded array, and the boundary / first interior line of u it is built from
def _side_lines(u, r):
    ny, nx = u.shape
    return ((np.s_[r:r + ny, r - 1], u[:, 0], u[:, 1]),
            (np.s_[r:r + ny, r + nx], u[:, -1], u[:, -2]),
            (np.s_[r - 1, r:r + nx], u[0, :], u[1, :]),
            (np.s_[r + ny, r:r + nx], u[-1, :], u[-2, :]))


def ghost_pad(u, radius: int, h: float, boundary, k_edges) -> np.ndarray:
    """Host copy of u embedded in a zero band of width `radius` with the first
    ghost layer closed per side (operators.py:44-75): Dirichlet 2 u_b - u_in,
    Sommerfeld u_in + (2ih k_b) u_b; ghost corners and deeper layers stay 0.
    The device kernels synthesise the same values on the fly (csrc/stencil.cuh);
    this copy serves LevelOperator.pad / halo_exchange callers."""
    u = np.asarray(u)
    ny, nx = u.shape
    pad = np.zeros((ny + 2 * radius, nx + 2 * radius), dtype=np.complex128)
    pad[radius:radius + ny, radius:radius + nx] = u
    two_ih = 2.0j * h
    for kind, kb, (where, ub, uin) in zip(boundary, k_edges, _side_lines(u, radius)):
        pad[where] = 2.0 * ub - uin if kind == DIRICHLET else uin + two_ih * kb * ub
    return pad


def ksq_ghost_pad(ksq, radius: int, boundary) -> np.ndarray:
    """k^2 with its ghost band: 2 k_b^2 - k_in^2 on Dirichlet sides, 0 elsewhere (operators.py:78-93)."""
    ksq = np.asarray(ksq, dtype=np.float64)
    ny, nx = ksq.shape
    pad = np.zeros((ny + 2 * radius, nx + 2 * radius))
    pad[radius:radius + ny, radius:radius + nx] = ksq
    for kind, (where, kb, kin) in zip(boundary, _side_lines(ksq, radius)):
        if kind == DIRICHLET:
            pad[where] = 2.0 * kb - kin
    return pad


class LevelOperator:
    """Matrix-free ``-Laplace - shift * I(k^2)`` on one grid level (GPU)."""

    def __init__(self, level, nx, ny, h, ksq, boundary, laplace: StencilKernel, mass: StencilKernel,
                 shift=1.0, level_scale=1.0, slab=None):
        if laplace.radius != mass.radius:
            raise ShapeError("laplace and mass kernels must share a radius")
        self.level = level
        self.nx, self.ny, self.h = int(nx), int(ny), float(h)
        # k^2 as a host array (the reference's form) or a CUDA float64 tensor from the
        # GPU-side setup (grid.build_hierarchy(device=True)); `ksq` then downloads on demand
        self._ksq_dev = None
        if dev.is_device(ksq):
            self._ksq_dev = dev.to_device(ksq, dtype="f8")
            self._ksq_host = None
        else:
            self._ksq_host = np.ascontiguousarray(ksq, dtype=np.float64)
        if tuple(ksq.shape) != (self.ny, self.nx):
            raise ShapeError(f"k^2 shape {tuple(ksq.shape)} != {(self.ny, self.nx)}")
        self.boundary = tuple(boundary)
        self.shift = complex(shift)
        self.radius = laplace.radius
        self.laplace, self.mass = laplace, mass
        # float conversion, once (operators.py:111-113)
        self.lap_coef = laplace.as_float() / self.h ** 2
        self.mass_coef = (-self.shift / level_scale) * mass.as_float().astype(np.complex128)
        self.slab = slab  # distributed.SlabSpec of this rank, None = whole grid
        self._handle = None
        self._kedges = None
        self._kpad = None

    @property
    def ksq(self) -> np.ndarray:
        if self._ksq_host is None:
            self._ksq_host = dev.to_host(self._ksq_dev)
        return self._ksq_host

    # host-side closure data of the reference object (operators.py:114-116), built on first use
    @property
    def k_edges(self):
        if self._kedges is None:
            kf = np.sqrt(self.ksq)
            self._kedges = (kf[:, 0], kf[:, -1], kf[0, :], kf[-1, :])
        return self._kedges

    @property
    def ksq_pad(self):
        if self._kpad is None:
            self._kpad = ksq_ghost_pad(self.ksq, self.radius, self.boundary)
        return self._kpad

    def pad(self, u) -> np.ndarray:
        """Ghost-padded host snapshot of u (operators.py:127-128)."""
        return ghost_pad(dev.to_host(u) if dev.is_device(u) else u, self.radius, self.h, self.boundary,
                         self.k_edges)

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
            if self.slab is None and self._ksq_dev is not None:
                check(L.hdb_op_create_dev(C.byref(h), self.nx, self.ny, self.radius, self.h, bc, f(lap), f(mre),
                                          f(mim), self._ksq_dev.data_ptr()))
            elif self.slab is None:
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
            sep = self.separable_factors()
            if sep is not None:
                sa, sm, lsc, msc = sep
                check(L.hdb_op_set_separable(h, f(sa), f(sm), lsc, msc.real, msc.imag))
        return self._handle

    def separable_factors(self):
        """(sa, sm, lsc, msc) with lap_coef = lsc (sa (x) sm + sm (x) sa) and
        mass_coef = msc (sm (x) sm), derived EXACTLY from the integer numerator
        tables (the Galerkin chain is a sum of tensor products),
        then checked in floating point to 2 ulp of the largest coefficient; None
        for radius 1 or a kernel pair without that structure (the device then
        uses the tap form)."""
        from fractions import Fraction
        if self.radius < 2:
            return None
        R, n = self.radius, 2 * self.radius + 1
        Mt, Lt = self.mass.numerators, self.laplace.numerators
        mu = [Mt[R][b] for b in range(n)]
        if mu[R] == 0 or any(Mt[a][b] * mu[R] != mu[a] * mu[b] for a in range(n) for b in range(n)):
            return None
        aR = Fraction(Lt[R][R], 2 * mu[R])
        al = [(Fraction(Lt[a][R]) - mu[a] * aR) / mu[R] for a in range(n)]
        if any(Lt[a][b] != al[a] * mu[b] + mu[a] * al[b] for a in range(n) for b in range(n)):
            return None
        sa = np.array([float(v) for v in al])
        sm = np.array([float(v) for v in mu])
        lsc = 1.0 / float(self.laplace.denominator) / self.h ** 2
        msc = complex(self.mass_coef[R, R]) / (sm[R] * sm[R])
        lap_r = lsc * (np.outer(sa, sm) + np.outer(sm, sa))
        mass_r = msc * np.outer(sm, sm)
        tol = 2.0 * np.finfo(float).eps
        if (np.abs(lap_r - self.lap_coef).max() > tol * np.abs(self.lap_coef).max()
                or np.abs(mass_r - self.mass_coef).max() > tol * np.abs(self.mass_coef).max()):
            return None
        return sa, sm, lsc, msc

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

    def residual_restrict(self, b, u, zero_mask=0):
        """Z^T (b - A u) in one pass (mg.py:116-117): the multigrid coarse right-hand
        side without storing the residual; bit-identical to ``residual`` followed by
        ``restrict_array``.  zero_mask: coarse Dirichlet sides to zero (bit 0 west,
        1 east, 2 south, 3 north).  Unsharded radius-1 operators."""
        host, (du, db) = self._io(u, b)
        ny, nx = self.shape
        dout = dev.empty(((ny - 1) // 2 + 1, (nx - 1) // 2 + 1))
        check(lib().hdb_op_residual_restrict(self.handle, db.data_ptr(), du.data_ptr(), dout.data_ptr(),
                                             int(zero_mask)))
        return dev.to_host(dout) if host else dout

    def jacobi_add(self, x, b, t, omega=0.8):
        """(Jacobi(x), Jacobi(x) + t) from one sweep: the last post-smoothing step with
        the A-DEF1 sum r + t folded in (mg.py:122, madp.py:327)."""
        host, (dx, db, dt) = self._io(x, b, t)
        dout, dsum = dev.empty(self.shape), dev.empty(self.shape)
        check(lib().hdb_op_jacobi_add(self.handle, dx.data_ptr(), db.data_ptr(), dout.data_ptr(), float(omega),
                                      dt.data_ptr(), dsum.data_ptr()))
        return (dev.to_host(dout), dev.to_host(dsum)) if host else (dout, dsum)

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


def level_ksq(hierarchy, level):
    """Level k^2 for an operator: the device tensor of a GPU-built hierarchy, else the host array."""
    dk = hierarchy.device_ksq_at(level) if getattr(hierarchy, "device_ksq", None) is not None else None
    return dk if dk is not None else hierarchy.ksq_at(level)


def _level_operator(hierarchy, level, shift, slab=None):
    lv = hierarchy.level(level)
    lap, mass = level_kernels(level)
    return LevelOperator(level, lv.nx, lv.ny, lv.h, level_ksq(hierarchy, level), hierarchy.boundary, lap, mass,
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


def _ghost_weights(kind, h, kb):
    """(boundary point, first interior point) weights that replace one ghost value."""
    if kind == DIRICHLET:
        return np.full(kb.shape, 2.0 + 0.0j), np.full(kb.shape, -1.0 + 0.0j)
    return 2.0j * h * kb, np.full(kb.shape, 1.0 + 0.0j)


def assemble_csr(op: LevelOperator, max_points: int = DEFAULT_ASSEMBLY_LIMIT):
    """The operator as an explicit scipy CSR matrix (operators.py:261-328), built
    from the stencil coefficients and the closure algebra, independently of the
    device kernels, so each can certify the other.  Host-side test oracle.

    Row p = j*nx + i.  Every tap (oj, oi) contributes coef = lap + mass * ksq_pad
    at the neighbour; a neighbour in the first ghost layer is redistributed onto
    the boundary point and the first interior point with the closure weights;
    anything further out is zero padding; Dirichlet rows are identity rows."""
    import scipy.sparse as sp
    from .errors import CapacityError
    if op.npoints > max_points:
        raise CapacityError(f"{op.npoints} points exceed the assembly guard {max_points}")
    nx, ny, r = op.nx, op.ny, op.radius
    J, I = np.divmod(np.arange(op.npoints), nx)
    free = np.ones(op.npoints, dtype=bool)
    for kind, hit in zip(op.boundary, (I == 0, I == nx - 1, J == 0, J == ny - 1)):
        if kind == DIRICHLET:
            free &= ~hit
    rows, cols, vals = [np.flatnonzero(~free)], [np.flatnonzero(~free)], [np.ones((~free).sum(), np.complex128)]
    P, Jf, If = np.flatnonzero(free), J[free], I[free]
    kw, ke, ks, kn = op.k_edges
    for oj in range(-r, r + 1):
        for oi in range(-r, r + 1):
            jj, ii = Jf + oj, If + oi
            coef = op.lap_coef[oj + r, oi + r] + op.mass_coef[oj + r, oi + r] * op.ksq_pad[jj + r, ii + r]
            nz = coef != 0
            xin, yin = (ii >= 0) & (ii < nx), (jj >= 0) & (jj < ny)
            m = nz & xin & yin
            rows.append(P[m]); cols.append(jj[m] * nx + ii[m]); vals.append(coef[m])
            # first ghost layer on each side: (mask, boundary index, interior index, k_b, side kind)
            ghosts = ((nz & yin & (ii == -1), lambda q: (jj[q], 0), lambda q: (jj[q], 1), lambda q: kw[jj[q]], 0),
                      (nz & yin & (ii == nx), lambda q: (jj[q], nx - 1), lambda q: (jj[q], nx - 2),
                       lambda q: ke[jj[q]], 1),
                      (nz & xin & (jj == -1), lambda q: (0, ii[q]), lambda q: (1, ii[q]), lambda q: ks[ii[q]], 2),
                      (nz & xin & (jj == ny), lambda q: (ny - 1, ii[q]), lambda q: (ny - 2, ii[q]),
                       lambda q: kn[ii[q]], 3))
            for mask, at_b, at_in, kb_of, side in ghosts:
                if not mask.any():
                    continue
                wb, wi = _ghost_weights(op.boundary[side], op.h, kb_of(mask))
                for (yy, xx), w in ((at_b(mask), wb), (at_in(mask), wi)):
                    rows.append(P[mask]); cols.append(np.broadcast_to(yy, mask.sum()) * nx + xx)
                    vals.append(coef[mask] * w)
    mat = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                        shape=(op.npoints, op.npoints))
    return mat.tocsr()


def assemble_dense(op: LevelOperator, max_points: int = 40_000) -> np.ndarray:
    """Dense form of assemble_csr (operators.py:331-333)."""
    return assemble_csr(op, max_points=max_points).toarray()


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
