"""ctypes binding of libhdb200.so (declarations: include/hdb200.h).

There is no CPU fallback: importing the package succeeds without a GPU (so the
host-side setup code and the C-ABI symbol table can be checked on a CPU box),
but every compute entry point calls ``lib()``, which raises ``DeviceError``
when the library is missing or no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigError, DeviceError, HelmdefError, MgDivergence, NumericalError, ShapeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhdb200.so")

LINOP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
ITER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_double)

vp, i32, i64, f64 = C.c_void_p, C.c_int, C.c_longlong, C.c_double
P = C.POINTER

# name -> argtypes (restype is always c_int status unless listed in _RESTYPE)
SIGNATURES = {
    "hdb_version": [],
    "hdb_last_error": [],
    "hdb_init": [i32],
    "hdb_stream": [P(vp)],
    "hdb_set_stream": [vp],
    "hdb_sync": [],
    "hdb_stats": [P(i64), P(i64)],
    "hdb_op_create": [P(vp), i32, i32, i32, f64, P(i32), P(f64), P(f64), P(f64), P(f64)],
    "hdb_op_destroy": [vp],
    "hdb_op_create_slab": [P(vp), i32, i32, i32, f64, P(i32), P(f64), P(f64), P(f64), P(f64), i32, i32, i32, i32,
                           P(i32), P(i32)],
    "hdb_comm_unique_id": [C.c_char_p],
    "hdb_comm_init_nccl": [C.c_char_p, i32, i32],
    "hdb_comm_init_threads": [i64, i32, i32],
    "hdb_comm_selftest_nccl": [],
    "hdb_plan_gather_rows": [P(i32), i32, i32, i32, P(i32), P(i32)],
    "hdb_thread_engine_begin": [i32],
    "hdb_thread_engine_end": [],
    "hdb_op_apply": [vp, vp, vp],
    "hdb_op_create_dev": [P(vp), i32, i32, i32, f64, P(i32), P(f64), P(f64), P(f64), vp],
    "hdb_setup_ksq_constant": [vp, i64, f64],
    "hdb_setup_ksq_wedge": [vp, i32, i32, f64, f64, f64, f64, f64, i32, P(f64)],
    "hdb_setup_ksq_raster": [vp, i32, i32, f64, f64, f64, f64, f64, vp, i32, i32, f64, f64, f64, f64],
    "hdb_setup_inject": [vp, i32, i32, vp],
    "hdb_setup_stats": [vp, i64, P(f64)],
    "hdb_setup_point_source": [vp, i64, i64, f64],
    "hdb_op_residual": [vp, vp, vp, vp],
    "hdb_op_resnorm": [vp, vp, vp, P(f64)],
    "hdb_op_jacobi": [vp, vp, vp, vp, f64],
    "hdb_op_residual_restrict": [vp, vp, vp, vp, i32],
    "hdb_op_jacobi_add": [vp, vp, vp, vp, f64, vp, vp],
    "hdb_restrict": [vp, i32, i32, vp, i32],
    "hdb_prolong": [vp, i32, i32, vp, vp],
    "hdb_dot": [vp, vp, i64, P(f64)],
    "hdb_mg_create": [P(vp), P(vp), i32, P(f64), i32, f64, i32, i32, f64, f64, i32],
    "hdb_mg_destroy": [vp],
    "hdb_mg_vcycle": [vp, vp, vp, vp],
    "hdb_fgmres": [i64, LINOP_FN, vp, LINOP_FN, vp, vp, vp, vp, f64, i32, ITER_FN, vp,
                   P(i32), P(f64), P(i32), P(f64), i32],
    "hdb_op_gmres": [vp, vp, vp, f64, i32, i32, P(i32), P(f64)],
    "hdb_bicgstab": [i64, LINOP_FN, vp, LINOP_FN, vp, vp, vp, vp, f64, i32, P(i32), P(f64), P(i32), P(f64), i32,
                     P(i32)],
    "hdb_resident_profile": [i32, P(i64)],
    "hdb_solver_create": [P(vp), i32, f64, i32],
    "hdb_solver_set_level": [vp, i32, vp, vp, vp, i32, f64, i32, f64, i32],
    "hdb_solver_solve": [vp, vp, vp, i32],
    "hdb_solver_report": [vp, P(i32), P(i32), P(f64), P(f64), P(i32)],
    "hdb_solver_history": [vp, P(f64), P(f64), i32],
    "hdb_solver_counts": [vp, i32, i32, P(i32), i32, P(i32)],
    "hdb_solver_matvecs": [vp, P(i64), i32],
    "hdb_solver_precond": [vp, i32, vp, vp],
    "hdb_solver_profile": [vp, P(f64), P(i64), i32, P(i64), P(i64)],
    "hdb_solver_bytes": [vp, P(f64)],
    "hdb_solver_destroy": [vp],
    "hdb_option": [C.c_char_p, i32],
    "hdb_op_set_separable": [vp, P(f64), P(f64), f64, f64, f64],
    "hdb_kprof": [i32],
    "hdb_kprof_read": [i32, C.c_char_p, P(i64), P(f64), P(f64)],
}
_RESTYPE = {"hdb_last_error": C.c_char_p}

_lock = threading.Lock()
_lib = None
_device = None


def load_library(path: str = LIB_PATH):
    """dlopen the library and declare every entry point (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"{path} is missing: build it with `python -m paper_2412_04980_b200._build`")
    lib = C.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def lib():
    """The library with a CUDA device selected; raises DeviceError otherwise."""
    global _device
    L = load_library()
    if _device is None:
        with _lock:
            if _device is None:
                dev = int(os.environ.get("HDB_DEVICE", "0"))
                try:
                    import torch
                    if torch.cuda.is_available():
                        dev = torch.cuda.current_device() if "HDB_DEVICE" not in os.environ else dev
                        torch.cuda.set_device(dev)
                except ImportError:
                    pass
                st = L.hdb_init(dev)
                if st != 0:
                    raise DeviceError(f"hdb_init({dev}) failed: {L.hdb_last_error().decode()}")
                # order library work on torch's current stream so device tensors
                # produced by torch are visible to the kernels without extra syncs
                try:
                    import torch
                    if torch.cuda.is_available():
                        check_raw(L, L.hdb_set_stream(torch.cuda.current_stream(dev).cuda_stream))
                except ImportError:
                    pass
                _device = dev
    return L


_STATUS = {1: ShapeError, 2: DeviceError, 3: NumericalError, 4: MgDivergence}
# 5 (Bi-CGSTAB breakdown) is raised by krylov.bicgstab itself (it carries the iterate)


def check_raw(L, status: int):
    if status != 0:
        raise DeviceError(L.hdb_last_error().decode())


def check(status: int):
    if status == 0:
        return
    msg = _lib.hdb_last_error().decode() if _lib is not None else "?"
    cls = _STATUS.get(status, HelmdefError)
    if status == 1 and ("preset" in msg or "config" in msg.lower()):
        cls = ConfigError
    raise cls(msg)


def kprof(enable: bool):
    """Arm (zero + per-launch CUDA events) or disarm the library's launch accounting."""
    check(lib().hdb_kprof(1 if enable else 0))


def kprof_read() -> dict:
    """{family: {"launches", "alg_bytes", "device_ms"}} since the last kprof(...)."""
    L = lib()
    cnt = C.c_longlong()
    check(L.hdb_kprof_read(-1, None, C.byref(cnt), C.byref(C.c_double()), C.byref(C.c_double())))
    out = {}
    for f in range(cnt.value):
        name = C.create_string_buffer(32)
        n, b, ms = C.c_longlong(), C.c_double(), C.c_double()
        check(L.hdb_kprof_read(f, name, C.byref(n), C.byref(b), C.byref(ms)))
        out[name.value.decode()] = {"launches": n.value, "alg_bytes": b.value, "device_ms": ms.value}
    return out


def device_index() -> int:
    lib()
    return _device


def stream_ptr() -> int:
    s = vp()
    check(lib().hdb_stream(C.byref(s)))
    return s.value or 0
