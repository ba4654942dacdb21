"""amgb200: B200-native solve phase of classical-AMG preconditioned CG.

Drop-in for the reference's hot path (``amgkit.krylov.pcg`` driving
``amgkit.hierarchy.vcycle``; see SURVEY.md 8 and DESIGN.md).  Setup stays in
the reference; its output is uploaded once::

    from amgkit import setup, AmgConfig                       # reference setup
    import paper_2102_07417_b200 as amgb200
    h = setup(A, AmgConfig(smoother="fsai"))
    dh = amgb200.DeviceHierarchy.from_reference(h)            # one upload
    res = amgb200.pcg(dh.A0, b, apply_m=dh.vcycle,
                      config=amgb200.KrylovConfig(rtol=1e-8))  # whole solve on the GPU

Several GPUs from one process: ``cl = amgb200.DeviceClique(h, devices=[0, 1])``
then ``amgb200.pcg(cl.A0, b, apply_m=cl.vcycle)``.

Reference names mirrored: ``pcg``, ``KrylovConfig``, ``KrylovResult``,
``vcycle``, ``spmv``, ``apply_smoother``, ``AmgError``,
``DimensionMismatchError``, ``NotSpdError``.
"""
from .errors import AmgError, BreakdownError, DimensionMismatchError, NotSpdError  # noqa: F401
from .device import DeviceHierarchy, DeviceMatrix, DeviceVcycle, model_bytes_flops  # noqa: F401
from .krylov import KrylovConfig, KrylovResult, bicgstab, pcg  # noqa: F401
from .clique import DeviceClique  # noqa: F401
from .ops import apply_smoother, coarse_solve, spmv, vcycle  # noqa: F401

__version__ = "0.1.0"
