"""Exception types of the device path, mirroring ``amgkit/errors.py``.

Names and hierarchy follow the reference (``AmgError`` base,
``DimensionMismatchError(op, left, right)``, ``NotSpdError``).  When the
reference package is importable the classes also derive from its types, so
code written against ``amgkit`` (``except amgkit.NotSpdError``) keeps working
unchanged with the device path.
"""
from __future__ import annotations

try:  # optional: make `except amgkit.X` catch ours
    from amgkit import errors as _ref  # type: ignore

    _RefAmg = (_ref.AmgError,)
    _RefDim = (_ref.DimensionMismatchError,)
    _RefSpd = (_ref.NotSpdError,)
    _RefBrk = (_ref.BreakdownError,)
except Exception:  # pragma: no cover - reference absent (GPU box)
    _RefAmg = _RefDim = _RefSpd = _RefBrk = ()


class AmgError(*(_RefAmg or (Exception,))):
    """Base class (``amgkit/errors.py:4-5``); also raised for CUDA / NCCL failures."""


class DimensionMismatchError(AmgError, *_RefDim):
    """Operands have incompatible shapes (``amgkit/errors.py:8-15``)."""

    def __init__(self, op, left, right):
        Exception.__init__(self, f"{op}: incompatible shapes {left} and {right}")
        self.op = op
        self.left = left
        self.right = right


class NotSpdError(AmgError, *_RefSpd):
    """Non-positive PCG curvature (``amgkit/errors.py:26-27``, ``krylov.py:67-72``)."""


class BreakdownError(AmgError, *_RefBrk):
    """BiCGstab breakdown (``amgkit/errors.py:30-31``, ``krylov.py:128-189``)."""
