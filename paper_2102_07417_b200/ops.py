"""Per-operation entry points with the reference's signatures.

* ``spmv(A, x)``                     -- ``amgkit/sparse.py:203-217``
* ``vcycle(h, y, level=0)``          -- ``amgkit/hierarchy.py:294-312``
* ``apply_smoother(sm, A, b, x0, steps)`` -- ``amgkit/smoothers.py:168-173``
* ``coarse_solve(h, b)``             -- ``AmgHierarchy.coarse_solve`` (``hierarchy.py:149-152``)

``A`` / ``h`` are device objects (:class:`DeviceMatrix`,
:class:`DeviceHierarchy`); host numpy vectors are copied in and out, CUDA
float64 tensors are used in place.
"""
from __future__ import annotations

from .device import DeviceHierarchy, DeviceMatrix, DeviceSmoother

__all__ = ["spmv", "vcycle", "apply_smoother", "coarse_solve"]


def spmv(A, x):
    if not isinstance(A, DeviceMatrix):
        raise TypeError("spmv: A must be a DeviceMatrix (no CPU fallback)")
    return A(x)


def vcycle(h, y, level=0):
    if not isinstance(h, DeviceHierarchy):
        raise TypeError("vcycle: h must be a DeviceHierarchy (no CPU fallback)")
    return h.apply_vcycle(y, level)


def apply_smoother(sm, A, b, x0, steps):
    """``sm``: ``dh.smoother(k)`` (or the level index, or None for A's level); ``A``: ``dh.matrix(k, "a")``."""
    if not isinstance(A, DeviceMatrix) or A.slot != "a":
        raise TypeError("apply_smoother: A must be the level operator DeviceMatrix")
    if isinstance(sm, DeviceSmoother):
        if sm.dh is not A.dh or sm.level != A.level:
            raise TypeError("apply_smoother: smoother and operator belong to different levels")
        level = sm.level
    else:
        level = A.level if sm is None else int(sm)
    return A.dh.apply_smoother(level, b, x0, steps)


def coarse_solve(h, b):
    if not isinstance(h, DeviceHierarchy):
        raise TypeError("coarse_solve: h must be a DeviceHierarchy")
    return h.coarse_solve(b)
