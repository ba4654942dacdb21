"""Replay of the reference's final FSAI row solves on the host (hierarchy loading only).

See ``csrc/fsai_host.c``: the coefficients of an FSAI factor G are a pure
function of the level operator A and G's final pattern
(``amgkit/smoothers.py:80-96``), computed with the LAPACK ``dpotrf`` /
``dpotrs`` that ``scipy.linalg.cho_factor`` / ``cho_solve`` use.  The function
addresses come from ``scipy.linalg.cython_lapack`` (scipy's own OpenBLAS), so
the replay executes the same routines as the reference's setup.  This is
setup data preparation for the frozen-hierarchy cache, not the solve path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import FSAI_LIB, build_fsai_host

__all__ = ["fsai_values"]

_lib = None
_fns = None


def _load():
    global _lib, _fns
    if _lib is None:
        if not os.path.exists(FSAI_LIB):
            build_fsai_host()
        _lib = ctypes.CDLL(FSAI_LIB)
        _lib.amgh_fsai_values.restype = ctypes.c_int64
        _lib.amgh_fsai_values.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64] + [ctypes.c_void_p] * 7 + [
            ctypes.c_int]
        import scipy.linalg.cython_lapack as cl

        get = ctypes.pythonapi.PyCapsule_GetPointer
        get.restype = ctypes.c_void_p
        get.argtypes = [ctypes.py_object, ctypes.c_char_p]
        name = ctypes.pythonapi.PyCapsule_GetName
        name.restype = ctypes.c_char_p
        name.argtypes = [ctypes.py_object]
        caps = cl.__pyx_capi__
        _fns = tuple(get(caps[f], name(caps[f])) for f in ("dpotrf", "dpotrs"))
    return _lib, _fns


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def fsai_values(a, g_offsets, g_cols, fallback_mask=None, threads=None, allow_failed=False):
    """Values of the FSAI factor with pattern (g_offsets, g_cols) for operator ``a``.

    ``fallback_mask[i]`` (uint8) marks rows the reference reset to the Jacobi
    row ``1/sqrt(a_ii)``.  Rows whose local Cholesky fails come back NaN; unless
    ``allow_failed`` that raises (the reference would have fallen back there).
    """
    lib, (potrf, potrs) = _load()
    offs = np.ascontiguousarray(g_offsets, dtype=np.int64)
    cols = np.ascontiguousarray(g_cols, dtype=np.int32)
    ao = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
    ac = np.ascontiguousarray(a.col_indices, dtype=np.int32)
    av = np.ascontiguousarray(a.values, dtype=np.float64)
    n = offs.size - 1
    if n != a.nrows:
        raise ValueError("pattern and operator disagree on the row count")
    if cols.size and (cols.min() < 0 or cols.max() >= a.ncols):
        raise ValueError("FSAI pattern column out of range")
    fb = None if fallback_mask is None else np.ascontiguousarray(fallback_mask, dtype=np.uint8)
    out = np.empty(cols.size, dtype=np.float64)
    nt = threads or min(64, os.cpu_count() or 1)
    r = lib.amgh_fsai_values(potrf, potrs, n, _ptr(ao), _ptr(ac), _ptr(av), _ptr(offs), _ptr(cols),
                             None if fb is None else _ptr(fb), _ptr(out), nt)
    if r < 0:
        raise ValueError(f"FSAI replay: row {-1 - r} is flagged as a Jacobi fallback but has off-diagonal entries")
    if r > 0 and not allow_failed:
        raise ValueError(f"FSAI replay: {r} rows lost positive definiteness (the reference fell back there)")
    return out
