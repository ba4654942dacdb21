"""Device PCG behind the reference's solver API (``amgkit/krylov.py``).

``pcg(apply_a, b, apply_m=None, x0=None, config=None) -> KrylovResult`` keeps
the reference signature, config and result types (``krylov.py:18-40``).
``apply_a`` must be a level-0 :class:`DeviceMatrix` and ``apply_m`` the
:class:`DeviceVcycle` of the same :class:`DeviceHierarchy`; the whole loop --
initial residual, every iteration, the periodic residual replacement and the
true-residual check at declared convergence -- then runs on the GPU as one
CUDA-graph while loop (``amg_pcg``).  Plain Python callables are rejected
with ``TypeError``: there is no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _capi as C
from .device import DeviceMatrix, DeviceVcycle

__all__ = ["KrylovConfig", "KrylovResult", "pcg", "bicgstab"]


@dataclass
class KrylovConfig:
    """``amgkit/krylov.py:18-23``."""

    rtol: float = 1e-8
    max_iters: int = 5000
    record_history: bool = False
    recompute_every: int = 50


@dataclass
class KrylovResult:
    """``amgkit/krylov.py:26-33`` (plus device timing in ``solve_ms``)."""

    x: np.ndarray
    converged: bool
    n_iterations: int
    relres: float
    history: list = field(default_factory=list)
    restarts: int = 0
    solve_ms: float = 0.0


def pcg(apply_a, b, apply_m=None, x0=None, config=None):
    """Preconditioned CG on the device (control flow of ``amgkit/krylov.py:40-92``).

    Raises :class:`NotSpdError` (message contains "curvature") on a
    non-positive curvature, exactly as the reference.
    """
    from .clique import _CliqueOp

    if isinstance(apply_a, _CliqueOp):
        if apply_a.kind != "A0" or not isinstance(apply_m, _CliqueOp) or apply_m.kind != "vcycle" or \
                apply_m.clique is not apply_a.clique:
            raise TypeError("pcg: a DeviceClique solve takes cl.A0 and cl.vcycle of the same clique")
        return apply_a.clique.pcg(b, x0=x0, config=config)
    if not isinstance(apply_a, DeviceMatrix) or apply_a.level != 0 or apply_a.slot != "a":
        raise TypeError("pcg: apply_a must be DeviceHierarchy.A0 (no CPU fallback)")
    if not isinstance(apply_m, DeviceVcycle) or apply_m.dh is not apply_a.dh:
        raise TypeError("pcg: apply_m must be the DeviceVcycle of the same DeviceHierarchy")
    cfg = config or KrylovConfig()
    dh = apply_a.dh
    n = dh.levels[0]["n"]
    bin_, dev = dh._vec_in(b, n, "pcg", (n, n))
    x0in = None
    if x0 is not None:
        x0in = dh._vec_in_like(x0, n, "pcg", (n, n), dev, bin_)
    x = dh._vec_out(bin_, n)
    n_iter = C.I32(0)
    relres = C.D(0.0)
    conv = C.I32(0)
    hist_len = C.I32(0)
    curv = C.D(0.0)
    hist = np.empty(cfg.max_iters + 1, dtype=np.float64) if cfg.record_history else None
    import ctypes

    st = C.lib().amg_pcg(
        dh._h, C.ptr(bin_), C.ptr(x0in), float(cfg.rtol), int(cfg.max_iters), int(cfg.recompute_every),
        C.ptr(x), ctypes.byref(n_iter), ctypes.byref(relres), ctypes.byref(conv),
        C.ptr(hist), ctypes.byref(hist_len), ctypes.byref(curv), dev,
    )
    C.check(st)
    history = []
    if hist is not None:
        history = [(i, float(hist[i])) for i in range(hist_len.value)]
    s = dh.stats()
    return KrylovResult(
        x=x,
        converged=bool(conv.value),
        n_iterations=int(n_iter.value),
        relres=float(relres.value),
        history=history,
        restarts=0,
        solve_ms=float(s["solve_ms"]),
    )


def bicgstab(apply_a, b, apply_m=None, x0=None, config=None):
    """Preconditioned BiCGstab on the device (control flow of ``amgkit/krylov.py:95-193``).

    Used by the reference for operator-filtered (nonsymmetric) hierarchies
    (``amgkit/cli.py:242-251``).  Raises :class:`BreakdownError` where the
    reference does.
    """
    import ctypes

    if not isinstance(apply_a, DeviceMatrix) or apply_a.level != 0 or apply_a.slot != "a":
        raise TypeError("bicgstab: apply_a must be DeviceHierarchy.A0 (no CPU fallback)")
    if not isinstance(apply_m, DeviceVcycle) or apply_m.dh is not apply_a.dh:
        raise TypeError("bicgstab: apply_m must be the DeviceVcycle of the same DeviceHierarchy")
    cfg = config or KrylovConfig()
    dh = apply_a.dh
    n = dh.levels[0]["n"]
    bin_, dev = dh._vec_in(b, n, "bicgstab", (n, n))
    x0in = None
    if x0 is not None:
        x0in = dh._vec_in_like(x0, n, "bicgstab", (n, n), dev, bin_)
    x = dh._vec_out(bin_, n)
    n_iter, conv, rst, hist_len = C.I32(0), C.I32(0), C.I32(0), C.I32(0)
    relres = C.D(0.0)
    hist = np.empty(cfg.max_iters + 1, dtype=np.float64) if cfg.record_history else None
    st = C.lib().amg_bicgstab(
        dh._h, C.ptr(bin_), C.ptr(x0in), float(cfg.rtol), int(cfg.max_iters), int(cfg.recompute_every),
        C.ptr(x), ctypes.byref(n_iter), ctypes.byref(relres), ctypes.byref(conv), ctypes.byref(rst),
        C.ptr(hist), ctypes.byref(hist_len), dev,
    )
    C.check(st)
    history = []
    if hist is not None:
        # the reference numbers history entries by iteration (restarts / s-exits keep the count)
        history = [(i, float(hist[i])) for i in range(hist_len.value)]
    return KrylovResult(x=x, converged=bool(conv.value), n_iterations=int(n_iter.value), relres=float(relres.value),
                        history=history, restarts=int(rst.value))
