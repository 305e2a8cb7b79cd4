"""Device buffers (PyTorch is used only to own CUDA memory and order streams).

Fields cross the API either as numpy arrays (host; copied in and out, the
reference's calling convention) or as torch CUDA complex128 tensors (zero
copy).  ``raw_view`` wraps a raw device pointer handed out by the library
(e.g. inside a Krylov callback) as a torch tensor without copying.
"""
from __future__ import annotations

import numpy as np

from ._lib import lib
from .errors import DeviceError


def torch_mod():
    try:
        import torch
    except ImportError as err:  # pragma: no cover
        raise DeviceError("PyTorch is required for device buffers") from err
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available: this package has no CPU fallback")
    lib()  # make sure the library and its stream are initialised
    return torch


def is_device(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def to_device(a, dtype="c16"):
    """numpy / torch -> contiguous torch CUDA tensor (complex128 or float64)."""
    torch = torch_mod()
    td = torch.complex128 if dtype == "c16" else torch.float64
    if is_device(a):
        return a.to(td).contiguous()
    npd = np.complex128 if dtype == "c16" else np.float64
    return torch.from_numpy(np.ascontiguousarray(a, dtype=npd)).to("cuda", non_blocking=False)


def empty(shape, dtype="c16"):
    torch = torch_mod()
    return torch.empty(shape, dtype=torch.complex128 if dtype == "c16" else torch.float64, device="cuda")


def zeros(shape):
    torch = torch_mod()
    return torch.zeros(shape, dtype=torch.complex128, device="cuda")


def to_host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def copy_to_host(t, out: np.ndarray) -> np.ndarray:
    """device tensor -> an existing host array (no new allocation); synchronous."""
    torch = torch_mod()
    torch.from_numpy(out).copy_(t.detach())
    return out


def ptr(t) -> int:
    return t.data_ptr()


class _CAI:
    __slots__ = ("__cuda_array_interface__",)

    def __init__(self, p, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<c16", "data": (int(p), False),
                                         "version": 3, "strides": None, "stream": None}


def raw_view(p, shape):
    """torch tensor aliasing device memory at address p (complex128, C order)."""
    torch = torch_mod()
    return torch.as_tensor(_CAI(p, shape), device="cuda")
