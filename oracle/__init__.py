"""CPU oracle for the PCG + AMG solve path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's solve-phase algorithm, used only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs, and only as the checker or the timed CPU
baseline -- never as the product path (the product path in
``paper_2102_07417_b200`` has no CPU fallback and fails loudly without its
CUDA library).

Parity pin: every function here is checked against golden vectors produced by
the reference itself (``amgkit`` imported in the build container by
``tools/make_golden.py``, committed under ``tests/golden/``), see
``tests/test_oracle.py``.  ``rowsum.c`` restates numpy's reduction order in
plain C and is pinned bit-for-bit against ``np.add.reduceat``.
"""
from .solve import (  # noqa: F401
    KrylovConfig,
    KrylovResult,
    NotSpdError,
    BreakdownError,
    bicgstab,
    DimensionMismatchError,
    apply_smoother,
    coarse_solve,
    pcg,
    row_segment_sums,
    smoother_apply,
    spmv,
    vcycle,
)
