"""ctypes binding of the C-ABI (include/mgb.h) and status -> exception mapping.

The extension is REQUIRED: importing the facade without ``libmgb.so`` raises,
and compute calls on a machine without a B200 raise RuntimeError from the
library's MGB_CUDA status.  There is no CPU fallback anywhere in the product.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MGB_LIB_PATH") or os.path.join(HERE, "libmgb.so")  # override: experiments only

MGB_OK, MGB_CONFIG, MGB_NUMERIC, MGB_NONCONVERGED, MGB_CONTRACT, MGB_SINGULAR, MGB_CUDA, MGB_NCCL = range(8)
NET_CONV, NET_FC = 0, 1

P = C.c_void_p
I = C.c_int
I64 = C.c_int64
D = C.c_double
PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int)

# name -> (restype, argtypes); keep in the order of include/mgb.h
SIGNATURES = {
    "mgb_version": (I, []),
    "mgb_last_error": (C.c_char_p, []),
    "mgb_last_pivot": (I, []),
    "mgb_device_info": (I, [I, PI, PI, PI]),
    "mgb_apply_stencil": (I, [I, I, I, I, P, P, P, P, P]),
    "mgb_restrict": (I, [I, I, I, P, P, P, P]),
    "mgb_prolong": (I, [I, I, I, P, P, P, P]),
    "mgb_galerkin_product": (I, [I, I, I, I, P, P, P, P, PI, P]),
    "mgb_smoother_apply": (I, [I, I, I, I, P, P, D, P, P, P]),
    "mgb_infer_kernels": (I, [I, I, I, P, P, I, I, P, I64, D, I, P, P]),
    "mgb_lu_factor": (I, [I, P, P, P]),
    "mgb_lu_solve": (I, [I, P, P, P, P, P]),
    "mgb_hier_build": (I, [I, I, I, I, D, P, I, P, I, P, C.POINTER(P)]),
    "mgb_hier_build_classed": (I, [I, I, I, I, D, P, I, P, C.POINTER(P)]),
    "mgb_hier_destroy": (None, [P]),
    "mgb_hier_depth": (I, [P, PI, PI]),
    "mgb_hier_level_info": (I, [P, I, PI, PI, PI, PI, PD]),
    "mgb_hier_stencil_points": (I, [P, I, PI]),
    "mgb_hier_level_uniformity": (I, [P, I, PI]),
    "mgb_hier_pass_kernel": (I, [P, I, I, PI]),
    "mgb_hier_get_operator": (I, [P, I, P]),
    "mgb_hier_get_kernels": (I, [P, I, P]),
    "mgb_hier_get_mask": (I, [P, I, P]),
    "mgb_hier_operator_planes": (I, [P, I, C.POINTER(P)]),
    "mgb_hier_set_storage": (I, [P, I, P]),
    "mgb_hier_storage_info": (I, [P, I, PI, PI]),
    "mgb_hier_set_fused": (I, [P, I]),
    "mgb_hier_set_passes": (I, [P, I64, I, I64]),
    "mgb_hier_set_stream_kernel": (I, [P, I]),
    "mgb_hier_set_conv_smoother": (I, [P, I, I, P, P, I, D, D]),
    "mgb_convolve": (I, [I, I, I, P, P, P, P, P]),
    "mgb_conv_smoother_apply": (I, [I, I, I, I, P, P, I, D, D, P, P, P, P]),
    "mgb_hier_equip_inferred": (I, [P, I, I, P, I64, D, I, P]),
    "mgb_hier_equip_jacobi": (I, [P, D, P]),
    "mgb_hier_set_kernels": (I, [P, I, I, P, I, D, P]),
    "mgb_coarse_solve": (I, [P, P, P, P]),
    "mgb_residual": (I, [P, I, P, P, P, P, P]),
    "mgb_smooth": (I, [P, P, I, P, P, I, P]),
    "mgb_restrict_residual": (I, [P, I, P, P, P, P]),
    "mgb_prolong_correct": (I, [P, I, P, P, P]),
    "mgb_work_create": (I, [P, C.POINTER(P)]),
    "mgb_work_destroy": (None, [P]),
    "mgb_vcycle": (I, [P, P, I, P, P, I, I, P]),
    "mgb_run_cycles": (I, [P, P, P, P, I, I, I, I, P, P]),
    "mgb_run_cycles_host": (I, [P, P, P, P, I, I, I, I, P, P]),
    "mgb_run_cycles_host_many": (I, [P, P, I, P, P, I, I, I, I, P, P]),
    "mgb_solve": (I, [P, P, P, P, I, I, D, I, PD, PI, PI, PI, PD, P]),
    "mgb_krylov": (I, [I, I, I, P, P, P, I, I, P, P, D, I, I, PD, PI, PI, PI, P]),
    "mgb_dd_nccl_unique_id": (I, [P]),
    "mgb_dd_create": (I, [P, I, I, I, P, I, C.POINTER(P)]),
    "mgb_dd_destroy": (None, [P]),
    "mgb_dd_info": (I, [P, I, PI, PI, PI]),
    "mgb_dd_set_rhs": (I, [P, I, P, P]),
    "mgb_dd_get_solution": (I, [P, I, P, P]),
    "mgb_dd_run_cycles": (I, [P, I, I, I, I, P, P]),
    "mgb_time_pass": (I, [P, P, I, I, I, P, P, I, PD, P]),
    "mgb_dd_set_exchange": (I, [P, P, P]),
    "mgb_dd_set_option": (I, [P, C.c_char_p, I]),
    "mgb_dd_stats": (I, [P, C.POINTER(I64), PI]),
    "mgb_ad_scratch_doubles": (I, [I]),
    "mgb_ad_axpby": (I, [I64, D, P, D, P, P, P]),
    "mgb_ad_mul": (I, [I64, P, P, I64, P, P]),
    "mgb_ad_leaky": (I, [I64, P, D, P, P, P]),
    "mgb_ad_sum_axis1": (I, [I64, I, I, P, P, P]),
    "mgb_ad_bcast_axis1": (I, [I64, I, I, P, P, P]),
    "mgb_ad_dot": (I, [I64, P, P, P, P, P]),
    "mgb_ad_stencil_adjoint": (I, [I, I, P, P, P, P, I, P, P]),
    "mgb_ad_pconv_kgrad": (I, [I, I, P, P, P, I, P, P]),
    "mgb_ad_conv_kgrad": (I, [I, I, I, P, P, P, P, I, P, P]),
    "mgb_ad_conv_batch": (I, [I64, I, P, P, P, P]),
    "mgb_ad_conv_batch_bwd": (I, [I64, I, P, P, P, P, I, P, I, P, P]),
    "mgb_ad_matmul": (I, [I, I, I, P, I, P, I, I, P, P, P]),
    "mgb_lu_solve_t": (I, [I, P, P, P, P, P, P]),
    "mgb_ad_adam": (I, [I64, P, P, P, P, D, D, D, D, I, P]),
    "mgb_guard_check": (I, [PI, PI]),
    "mgb_last_launch_count": (I64, [P]),
}

_lib = None


def lib():
    """Load libmgb.so (built in-tree by build.py); raise loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -m paper_2102_12071_b200.build); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int):
    """Map an mgb_status onto the reference's exception classes (errors.py)."""
    if status == MGB_OK:
        return
    L = lib()
    msg = L.mgb_last_error().decode(errors="replace")
    if status == MGB_CONFIG:
        raise errors.ConfigError(msg)
    if status == MGB_NUMERIC:
        raise errors.NumericError(msg)
    if status == MGB_NONCONVERGED:
        raise errors.NonConvergedError(msg)
    if status == MGB_CONTRACT:
        raise errors.ContractError(msg)
    if status == MGB_SINGULAR:
        raise errors.SingularMatrixError(msg, pivot_index=L.mgb_last_pivot())
    raise RuntimeError(f"mgb status {status}: {msg}")


def call(name, *args):
    check(getattr(lib(), name)(*args))
