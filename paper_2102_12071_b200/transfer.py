"""Full-coarsening grid transfers and the Galerkin product — facade over the
B200 kernels (reference transfer.py:28-222).

Coarse point c sits at fine index 2c + 1, rows_c = rows // 2; restriction is
full weighting FW/16 and prolongation twice that (half of bilinear), so the
materialised R equals 0.5 P^T.  Red-black coarsening is not on the B200 path
(no configuration uses it)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, device as dv
from .errors import ConfigError, ContractError, UnsupportedOperationError
from .grid import GridFunction, GridSpec, StencilField

FULL_WEIGHTING = np.array([[1.0, 2.0, 1.0],
                           [2.0, 4.0, 2.0],
                           [1.0, 2.0, 1.0]]) / 16.0


@dataclass(frozen=True)
class TransferPair:
    """transfer.py:39-47 (restriction/prolongation held as 3x3 tables)."""
    scheme: str
    fine: GridSpec
    coarse: GridSpec
    restriction: np.ndarray
    prolongation: np.ndarray
    stride: int
    offset: int


def coarsen_full(fine: GridSpec) -> TransferPair:
    """transfer.py:50-61."""
    rows_c, cols_c = fine.rows // 2, fine.cols // 2
    if rows_c < 1 or cols_c < 1:
        raise ConfigError(f"{fine.rows}x{fine.cols} grid cannot be coarsened further")
    mask_c = fine.mask[1::2, 1::2][:rows_c, :cols_c].copy()
    if not mask_c.any():
        raise ConfigError("coarsening left no active points")
    coarse = GridSpec(rows_c, cols_c, 2.0 * fine.spacing, mask_c)
    return TransferPair("full", fine, coarse, FULL_WEIGHTING.copy(), 2.0 * FULL_WEIGHTING, 2, 1)


def coarsen_checker(fine: GridSpec):
    raise UnsupportedOperationError("red-black coarsening is not on the B200 path")


coarsen_derotate = coarsen_checker


def _check_full(tp: TransferPair):
    if tp.scheme != "full":
        raise UnsupportedOperationError("only full coarsening runs on the B200 path")


def restrict(tp: TransferPair, u_fine: GridFunction) -> GridFunction:
    """transfer.py:108-121 (mgb_restrict)."""
    _check_full(tp)
    if u_fine.spec != tp.fine:
        raise ContractError("restrict: grid function not on the fine spec")
    x = dv.to_dev(u_fine.values)
    out = dv.empty((tp.coarse.rows, tp.coarse.cols))
    m = dv.mask_dev(tp.coarse.mask)
    _lib.call("mgb_restrict", 1, tp.fine.rows, tp.fine.cols, dv.ptr(m), dv.ptr(x), dv.ptr(out),
              dv.stream(out))
    return GridFunction(tp.coarse, dv.host(out))


def prolong(tp: TransferPair, u_coarse: GridFunction) -> GridFunction:
    """transfer.py:124-147 (mgb_prolong)."""
    _check_full(tp)
    if u_coarse.spec != tp.coarse:
        raise ContractError("prolong: grid function not on the coarse spec")
    x = dv.to_dev(u_coarse.values)
    out = dv.empty((tp.fine.rows, tp.fine.cols))
    m = dv.mask_dev(tp.fine.mask)
    _lib.call("mgb_prolong", 1, tp.fine.rows, tp.fine.cols, dv.ptr(m), dv.ptr(x), dv.ptr(out),
              dv.stream(out))
    return GridFunction(tp.fine, dv.host(out))


def galerkin_product(A: StencilField, tp: TransferPair) -> StencilField:
    """transfer.py:150-209 + _trim :212-222 (mgb_galerkin_product)."""
    _check_full(tp)
    if A.spec != tp.fine:
        raise ContractError("galerkin_product: operator not on the fine spec")
    if A.k != 3:
        raise UnsupportedOperationError("galerkin_product on the B200 path takes 3x3 stencils")
    Ad = dv.to_dev(A.data)
    out = dv.empty((tp.coarse.rows, tp.coarse.cols, 3, 3))
    mf = dv.mask_dev(tp.fine.mask)
    mc = dv.mask_dev(tp.coarse.mask)
    import ctypes as C
    k = C.c_int(0)
    _lib.call("mgb_galerkin_product", 1, tp.fine.rows, tp.fine.cols, 3, dv.ptr(Ad), dv.ptr(mf), dv.ptr(mc),
              dv.ptr(out), C.byref(k), dv.stream(out))
    data = dv.host(out)
    if k.value == 1:
        data = np.ascontiguousarray(data[:, :, 1:2, 1:2])
    return StencilField(tp.coarse, data)
