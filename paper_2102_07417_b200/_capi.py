"""ctypes binding of ``libamgb200.so`` (declared in ``include/amgb200.h``).

The library is built in-tree by ``paper_2102_07417_b200.build.build()``.
There is no CPU fallback: if the library is missing or no GPU is usable,
loading / handle creation raises :class:`AmgError`.
"""
from __future__ import annotations

import ctypes
import os

from .errors import AmgError, BreakdownError, DimensionMismatchError, NotSpdError

LIB_PATH = os.environ.get("AMGB200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libamgb200.so")

AMG_OK, AMG_E_ARG, AMG_E_DIM, AMG_E_NOT_SPD, AMG_E_CUDA, AMG_E_NCCL, AMG_E_STATE, AMG_E_BREAKDOWN = range(8)
AMG_A, AMG_P, AMG_PT, AMG_G, AMG_GT = range(5)
SLOT = {"a": AMG_A, "p": AMG_P, "pt": AMG_PT, "g": AMG_G, "gt": AMG_GT}
AMG_SMOOTHER_FSAI, AMG_SMOOTHER_JACOBI = 0, 1
AMG_COARSE_CHOLESKY, AMG_COARSE_LU = 0, 1

# every symbol the header declares (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "amg_create", "amg_destroy", "amg_last_error", "amg_get_version", "amg_set_levels",
    "amg_set_partition", "amg_upload_matrix", "amg_set_smoother", "amg_upload_coarse",
    "amg_set_cycle", "amg_finalize", "amg_local_rows", "amg_spmv", "amg_smoother",
    "amg_coarse_solve", "amg_vcycle", "amg_vcycle_level", "amg_pcg", "amg_get_stats", "amg_set_option", "amg_time_spmv",
    "amg_nccl_unique_id", "amg_set_halo", "amg_set_agglomeration", "amg_bicgstab",
    "amg_matrix_layout", "amg_matrix_bytes",
    "amg_device_galerkin", "amg_device_transpose", "amg_csr_result_shape", "amg_csr_result_fetch",
    "amg_csr_result_free",
)


class Stats(ctypes.Structure):
    _fields_ = [
        ("solve_ms", ctypes.c_double),
        ("e2e_ms", ctypes.c_double),
        ("launches_per_iter", ctypes.c_int64),
        ("launches_last", ctypes.c_int64),
        ("bytes_per_iter", ctypes.c_int64),
        ("flops_per_iter", ctypes.c_int64),
        ("graph_mode", ctypes.c_int),
        ("n_levels", ctypes.c_int),
        ("tail_level", ctypes.c_int),
        ("cluster", ctypes.c_int),
    ]


_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
D = ctypes.c_double


def lib():
    """Load (once) and return the library; raises AmgError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise AmgError(
            f"{LIB_PATH} not found: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
        )
    if "AMGB200_NCCL" not in os.environ:
        # multi-GPU: share torch's NCCL build (the one torch.distributed uses) rather than
        # whatever libnccl.so.2 the loader would find first (csrc/halo.h)
        try:
            import importlib.util

            spec = importlib.util.find_spec("nvidia.nccl")
            for root in (spec.submodule_search_locations or []) if spec else []:
                cand = os.path.join(root, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["AMGB200_NCCL"] = cand
                    break
        except Exception:
            pass
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "amg_create": (I32, [I32, I32, I32, P, ctypes.POINTER(P)]),
        "amg_destroy": (None, [P]),
        "amg_last_error": (ctypes.c_char_p, []),
        "amg_get_version": (I32, []),
        "amg_set_levels": (I32, [P, I32]),
        "amg_set_partition": (I32, [P, I32, P]),
        "amg_upload_matrix": (I32, [P, I32, I32, I64, I64, P, P, P]),
        "amg_set_smoother": (I32, [P, I32, I32, D, P, I64]),
        "amg_upload_coarse": (I32, [P, I32, P, I32, P]),
        "amg_set_cycle": (I32, [P, I32, I32]),
        "amg_finalize": (I32, [P]),
        "amg_local_rows": (I64, [P, I32]),
        "amg_spmv": (I32, [P, I32, I32, P, P, I32]),
        "amg_smoother": (I32, [P, I32, P, P, P, I32, I32]),
        "amg_coarse_solve": (I32, [P, P, P, I32]),
        "amg_vcycle": (I32, [P, P, P, I32]),
        "amg_vcycle_level": (I32, [P, I32, P, P, I32]),
        "amg_pcg": (I32, [P, P, P, D, I32, I32, P, P, P, P, P, P, P, I32]),
        "amg_get_stats": (I32, [P, ctypes.POINTER(Stats)]),
        "amg_set_option": (I32, [P, ctypes.c_char_p, I64]),
        "amg_time_spmv": (I32, [P, I32, I32, I32, ctypes.POINTER(D)]),
        "amg_nccl_unique_id": (I32, [P]),
        "amg_set_halo": (I32, [P, I32, I32, I64, I64, I32, P, P, I32, P, P, P]),
        "amg_set_agglomeration": (I32, [P, I32]),
        "amg_bicgstab": (I32, [P, P, P, D, I32, I32, P, P, P, P, P, P, P, I32]),
        "amg_matrix_layout": (I32, [P, I32, I32, ctypes.POINTER(I32)]),
        "amg_matrix_bytes": (I32, [P, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "amg_device_galerkin": (I32, [I32, I64, I64, P, P, P, P, P, P, I32, ctypes.POINTER(P)]),
        "amg_device_transpose": (I32, [I32, I64, I64, P, P, P, ctypes.POINTER(P)]),
        "amg_csr_result_shape": (I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "amg_csr_result_fetch": (I32, [P, P, P, P]),
        "amg_csr_result_free": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status, what=""):
    """Map a C status to the reference's exception types."""
    if status == AMG_OK:
        return
    msg = lib().amg_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == AMG_E_NOT_SPD:
        raise NotSpdError(msg)
    if status == AMG_E_BREAKDOWN:
        raise BreakdownError(msg)
    if status == AMG_E_DIM:
        err = DimensionMismatchError(what or "amgb200", "?", "?")
        err.args = (msg,)
        raise err
    raise AmgError(msg)


def ptr(a):
    """Raw data pointer of a contiguous numpy array or a CUDA torch tensor."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)
