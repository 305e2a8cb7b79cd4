"""Higher-order transfers Z^T / Z on the GPU (drop-in for reference transfers.py:59-111).

Kernels: csrc/kernels_transfer.cu (bit-identical to the reference's 25 strided
numpy passes).  numpy in -> numpy out; torch CUDA tensor in -> tensor out.
"""
from __future__ import annotations

import numpy as np

from . import device as dev
from ._lib import check, lib
from .errors import LevelError, ShapeError
from .grid import ComplexField

__all__ = ["restrict_array", "prolong_array", "restrict", "prolong", "coarse_size"]


def coarse_size(n: int) -> int:
    if (n - 1) % 2:
        raise LevelError(f"cannot coarsen {n} points: n-1 must be even")
    return (n - 1) // 2 + 1


def restrict_array(fine, zero_mask: int = 0):
    ny, nx = fine.shape
    ncy, ncx = coarse_size(ny), coarse_size(nx)
    host = not dev.is_device(fine)
    df = dev.to_device(fine)
    out = dev.empty((ncy, ncx))
    check(lib().hdb_restrict(df.data_ptr(), ny, nx, out.data_ptr(), int(zero_mask)))
    return dev.to_host(out) if host else out


def prolong_array(coarse, fine_shape: tuple, base=None):
    nfy, nfx = fine_shape
    ncy, ncx = coarse.shape
    if nfx != 2 * ncx - 1 or nfy != 2 * ncy - 1:
        raise ShapeError(f"fine shape {fine_shape} does not refine {tuple(coarse.shape)}")
    host = not dev.is_device(coarse)
    dc = dev.to_device(coarse)
    db = dev.to_device(base) if base is not None else None
    out = dev.empty((nfy, nfx))
    check(lib().hdb_prolong(dc.data_ptr(), nfy, nfx, db.data_ptr() if db is not None else None, out.data_ptr()))
    return dev.to_host(out) if host else out


def restrict(field, hierarchy):
    lvl = field.level
    if lvl + 1 > hierarchy.ml:
        raise LevelError(f"hierarchy has no level {lvl + 1}")
    data = restrict_array(field.grid_view(hierarchy))
    return ComplexField(level=lvl + 1, data=np.asarray(data).ravel())


def prolong(field, hierarchy):
    lvl = field.level
    if lvl - 1 < 1:
        raise LevelError("already at the finest level")
    fine = hierarchy.levels[lvl - 2]
    data = prolong_array(field.grid_view(hierarchy), (fine.ny, fine.nx))
    return ComplexField(level=lvl - 1, data=np.asarray(data).ravel())
