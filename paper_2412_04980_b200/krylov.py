"""Flexible GMRES / GMRES on the GPU (drop-in for reference krylov.py:31-182, 279-283).

The Arnoldi process runs in the CUDA library (csrc/engine.cu): fused MGS
launches (one per Hessenberg coefficient), deterministic device reductions,
one device->host read of the Hessenberg column per iteration, Givens
rotations and the least-squares update on the host (as in the reference).

``apply_A`` / ``apply_M`` may be:
  * a GPU ``LevelOperator.apply`` bound method, a ``CslpMultigrid.vcycle``
    bound method, or any object with a ``_device_apply(in_ptr, out_ptr)``
    method -> called on device buffers directly;
  * any other callable -> called with arrays of ``b``'s kind (numpy in,
    numpy out for numpy ``b``; torch CUDA tensors for a CUDA ``b``).
``dot`` (krylov.py:57-61): the Krylov engine computes every inner product on
the device with the library's deterministic conj-first reduction, which is
the contract of the reference's choices for it (np.vdot, the default, and
reduce_dot, parallel.py:168-195: conj(u).v, independent of the worker count).
Those, and this package's reduce_dot, are accepted; any other callable would
be silently replaced, so it is rejected with ConfigError instead.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import device as dev
from ._lib import ITER_FN, LINOP_FN, check, lib

__all__ = ["StopRule", "KrylovReport", "fgmres", "gmres", "bicgstab", "cslp_iteration_cap", "device_callable"]


@dataclass(frozen=True)
class StopRule:
    """Relative tolerance plus iteration cap (tol >= 1 => exactly one iteration)."""

    rel_tol: float
    max_iters: int

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.rel_tol < 0:
            raise ValueError("rel_tol must be nonnegative")


@dataclass
class KrylovReport:
    iterations: int
    final_relres: float
    residual_history: list = field(default_factory=list)
    converged: bool = False


def cslp_iteration_cap(level_size: int, c_it: float = 6.0) -> int:
    """ceil(c_it * N**(1/4)) (krylov.py:279-283)."""
    if level_size < 1:
        raise ValueError("level size must be >= 1")
    return int(math.ceil(c_it * float(level_size) ** 0.25 - 1e-9))


def device_callable(fn):
    """Return f(in_ptr, out_ptr) running on device buffers, or None."""
    obj = getattr(fn, "__self__", None)
    name = getattr(fn, "__name__", "")
    if obj is not None and hasattr(obj, "_device_apply") and name in ("apply", "vcycle", "_device_apply"):
        return obj._device_apply
    if hasattr(fn, "_device_apply"):
        return fn._device_apply
    return None


class _Bridge:
    """ctypes callback adapter that records the first Python exception."""

    def __init__(self, fn, shape, host: bool):
        self.fn, self.shape, self.host = fn, shape, host
        self.dfn = device_callable(fn) if fn is not None else None
        self.error = None
        self.cfunc = LINOP_FN(self._call)

    def _call(self, _user, pin, pout):
        try:
            if self.dfn is not None:
                self.dfn(pin, pout)
                return 0
            vin = dev.raw_view(pin, self.shape)
            vout = dev.raw_view(pout, self.shape)
            if self.host:
                res = self.fn(vin.cpu().numpy())
                vout.copy_(dev.to_device(np.asarray(res, dtype=np.complex128).reshape(self.shape)))
            else:
                res = self.fn(vin.clone())
                vout.copy_(res.reshape(self.shape))
            return 0
        except BaseException as err:  # noqa: BLE001 - re-raised after the C call
            if self.error is None:
                self.error = err
            return 1


def _check_dot(dot):
    """Accept only inner products the device reduction implements (see module doc)."""
    if dot is None or dot is np.vdot:
        return
    name = getattr(dot, "__name__", "")
    mod = getattr(dot, "__module__", "") or ""
    if name == "reduce_dot" and (mod.endswith(".parallel") or mod == "parallel"):
        return   # this package's or the reference's deterministic block dot
    from .errors import ConfigError
    raise ConfigError(f"custom dot {dot!r} is not supported: Krylov inner products run on the device "
                      "(conj-first deterministic reduction); pass dot=None, np.vdot or reduce_dot")


def fgmres(apply_A, apply_M, b, stop: StopRule, x0=None, dot=None, on_iteration=None):
    """Right-preconditioned flexible GMRES without restarts (krylov.py:61-177)."""
    _check_dot(dot)
    host = not dev.is_device(b)
    shape = tuple(b.shape)
    db = dev.to_device(b)
    dx = dev.empty(shape)
    dx0 = dev.to_device(x0) if x0 is not None else None
    A = _Bridge(apply_A, shape, host)
    M = _Bridge(apply_M, shape, host) if apply_M is not None else None
    hook_err = []

    def _hook(_u, it, rel):
        try:
            on_iteration(it, rel)
            return 0
        except BaseException as err:  # noqa: BLE001
            hook_err.append(err)
            return 1

    hook = ITER_FN(_hook) if on_iteration is not None else ITER_FN()
    cap = stop.max_iters + 1
    hist = (C.c_double * cap)()
    its, fin, conv = C.c_int(), C.c_double(), C.c_int()
    st = lib().hdb_fgmres(db.numel(), A.cfunc, None, M.cfunc if M else LINOP_FN(), None, db.data_ptr(),
                          dx0.data_ptr() if dx0 is not None else None, dx.data_ptr(), float(stop.rel_tol),
                          int(stop.max_iters), hook, None, C.byref(its), C.byref(fin), C.byref(conv), hist, cap)
    for err in (A.error, M.error if M else None, hook_err[0] if hook_err else None):
        if err is not None:
            raise err
    check(st)
    history = list(hist[: min(its.value + 1, cap)])
    rep = KrylovReport(its.value, fin.value, history, bool(conv.value))
    return (dev.to_host(dx) if host else dx), rep


def gmres(apply_A, apply_M, b, stop: StopRule, x0=None, dot=None, on_iteration=None):
    """GMRES with a fixed right preconditioner (same engine as fgmres)."""
    return fgmres(apply_A, apply_M, b, stop, x0=x0, dot=dot, on_iteration=on_iteration)


def bicgstab(apply_A, apply_M, b, stop: StopRule, x0=None, dot=None):
    """Right-preconditioned Bi-CGSTAB (krylov.py:185-276).  Raises BreakdownError
    carrying the best iterate and its report when rho or omega vanish."""
    from .errors import BreakdownError
    _check_dot(dot)
    host = not dev.is_device(b)
    shape = tuple(b.shape)
    db = dev.to_device(b)
    dx = dev.empty(shape)
    dx0 = dev.to_device(x0) if x0 is not None else None
    A = _Bridge(apply_A, shape, host)
    M = _Bridge(apply_M, shape, host) if apply_M is not None else None
    cap = stop.max_iters + 2
    hist = (C.c_double * cap)()
    its, fin, conv, hl = C.c_int(), C.c_double(), C.c_int(), C.c_int()
    st = lib().hdb_bicgstab(db.numel(), A.cfunc, None, M.cfunc if M else LINOP_FN(), None, db.data_ptr(),
                            dx0.data_ptr() if dx0 is not None else None, dx.data_ptr(), float(stop.rel_tol),
                            int(stop.max_iters), C.byref(its), C.byref(fin), C.byref(conv), hist, cap, C.byref(hl))
    for err in (A.error, M.error if M else None):
        if err is not None:
            raise err
    x = dev.to_host(dx) if host else dx
    rep = KrylovReport(its.value, fin.value, list(hist[: min(hl.value, cap)]), bool(conv.value))
    if st == 5:
        raise BreakdownError(lib().hdb_last_error().decode(), x=x, report=rep)
    check(st)
    return x, rep
