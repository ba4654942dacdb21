"""Device-backed ``run_solve`` and report, mirroring the reference caller.

* :func:`run_solve` follows ``amgkit/cli.py:237-295``: validate the method
  (pcg needs a symmetric hierarchy: operator filtering is rejected exactly as
  ``cli.py:242-251`` does), set the hierarchy up with the REFERENCE's
  ``amgkit.setup`` (or take a frozen one), then solve -- on the GPU, through
  :func:`krylov.pcg` / :func:`krylov.bicgstab` -- with the residual history.
* :class:`SolveReport` has the fields of ``amgkit/hierarchy.py:360-378``;
  :func:`report_emit` renders text / json (schema_version 1) / csv exactly as
  ``cli.py:296-342``.
* ``python -m paper_2102_07417_b200 solve ...`` exits 0 converged, 2 not
  converged, 1 on error (``cli.py:441-446, 499``).
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass

import numpy as np

from .errors import AmgError

__all__ = ["SolveReport", "run_solve", "report_emit", "level_table", "complexities", "DEFAULTS", "main"]

# the solve-relevant keys of the reference's CONFIG_KEYS (cli.py:38-73) with their defaults
DEFAULTS = {
    "solver.method": "pcg",
    "solver.rtol": 1e-8,
    "solver.max_iters": 5000,
    "solver.rhs_seed": 42,
    "interp.filter_rho": 1.0,
    "interp.filter_target": "none",
}

REPORT_SCALARS = (
    "method", "converged", "n_iterations", "rtol", "final_relres", "c_gd", "c_op", "n_levels",
    "matrix_n", "matrix_nnz", "setup_seconds", "solve_seconds", "total_seconds",
)


@dataclass
class SolveReport:
    """Fields of ``amgkit.hierarchy.SolveReport`` (``hierarchy.py:360-378``)."""

    method: str
    converged: bool
    n_iterations: int
    rtol: float
    final_relres: float
    c_gd: float
    c_op: float
    n_levels: int
    levels: list
    setup_seconds: float
    solve_seconds: float
    total_seconds: float
    matrix_n: int
    matrix_nnz: int
    history: list | None = None


def complexities(h):
    """(grid, operator) complexity; ``amgkit/hierarchy.py:315-321``."""
    n0 = h.levels[0].a.nrows
    nnz0 = max(h.levels[0].a.nnz, 1)
    return (sum(l.a.nrows for l in h.levels) / max(n0, 1), sum(l.a.nnz for l in h.levels) / nnz0)


def level_table(h):
    """Per-level summary; ``amgkit/hierarchy.py:324-341``."""
    rows, prev = [], None
    for k, l in enumerate(h.levels):
        n, nnz = l.a.nrows, l.a.nnz
        rows.append({"level": k, "n": n, "nnz": nnz, "avg_nnz_per_row": round(nnz / max(n, 1), 3),
                     "coarsening_ratio": round(n / prev, 4) if prev else 1.0})
        prev = n
    return rows


def run_solve(a, b, cfg=None, coords=None, hierarchy=None, device=0, options=None, devices=None):
    """Set up (reference) and solve (device); returns ``(result, report, hierarchy)``.

    ``devices`` (a list of GPU ids, PCG only): the rows are partitioned over
    those GPUs in this one process (:class:`clique.DeviceClique`).
    """
    from . import krylov
    from .device import DeviceHierarchy

    c = dict(DEFAULTS)
    c.update(cfg or {})
    method = str(c["solver.method"]).lower()
    if method not in ("pcg", "bicgstab"):
        raise AmgError(f"unknown solver {method!r} (pcg or bicgstab)")
    if (method == "pcg" and str(c["interp.filter_target"]).replace("-", "_") in ("operator", "both")
            and float(c["interp.filter_rho"]) < 1.0):
        raise AmgError("operator filtering can leave the coarse operators nonsymmetric, so conjugate gradients "
                       "cannot be trusted; use solver.method = bicgstab or filter the prolongation only")
    t0 = time.perf_counter()
    h = hierarchy
    if h is None:
        try:
            from amgkit.cli import _amg_config, load_config  # the reference's own setup path
            from amgkit.hierarchy import setup
        except Exception as exc:  # pragma: no cover - depends on the environment
            raise AmgError("run_solve: hierarchy setup needs the reference package (amgkit) or a frozen "
                           "hierarchy (hiercache.load_hierarchy)") from exc
        full = load_config()
        full.update({k: v for k, v in c.items() if k in full})
        h = setup(a, _amg_config(full, coords=coords))
    t1 = time.perf_counter()
    if devices is not None and len(devices) > 1:
        if method != "pcg":
            raise AmgError("run_solve: multi-GPU solves are PCG only")
        from .clique import DeviceClique

        dh = DeviceClique(h, devices, options=options)
    else:
        dh = DeviceHierarchy.from_reference(h, device=device if not devices else devices[0], options=options)
    kcfg = krylov.KrylovConfig(rtol=float(c["solver.rtol"]), max_iters=int(c["solver.max_iters"]),
                               record_history=True)
    solver = krylov.pcg if method == "pcg" else krylov.bicgstab
    t2 = time.perf_counter()
    result = solver(dh.A0, b, apply_m=dh.vcycle, config=kcfg)
    t3 = time.perf_counter()
    dh.close()
    c_gd, c_op = complexities(h)
    report = SolveReport(
        method=method, converged=bool(result.converged), n_iterations=int(result.n_iterations),
        rtol=float(c["solver.rtol"]), final_relres=float(result.relres), c_gd=round(c_gd, 6), c_op=round(c_op, 6),
        n_levels=len(h.levels), levels=level_table(h), setup_seconds=round(t1 - t0, 6),
        solve_seconds=round(t3 - t2, 6), total_seconds=round(t3 - t0, 6), matrix_n=int(h.levels[0].a.nrows),
        matrix_nnz=int(h.levels[0].a.nnz), history=[(int(i), float(r)) for i, r in result.history],
    )
    return result, report, h


def report_emit(report, fmt="text"):
    """Render a report as text, json, or csv (``amgkit/cli.py:313-342``)."""
    if fmt == "json":
        doc = {"schema_version": 1}
        for k in REPORT_SCALARS:
            doc[k] = getattr(report, k)
        doc["levels"] = report.levels
        return json.dumps(doc, indent=2) + "\n"
    if fmt == "csv":
        lines = ["level,n,nnz,avg_nnz_per_row,coarsening_ratio"]
        for row in report.levels:
            lines.append(f"{row['level']},{row['n']},{row['nnz']},{row['avg_nnz_per_row']},{row['coarsening_ratio']}")
        return "\n".join(lines) + "\n"
    if fmt == "text":
        lines = [f"{k:>16}: {getattr(report, k)}" for k in REPORT_SCALARS]
        lines.append(f"{'level':>5} {'n':>10} {'nnz':>12} {'nnz/row':>9} {'ratio':>7}")
        for row in report.levels:
            lines.append(f"{row['level']:>5} {row['n']:>10} {row['nnz']:>12} "
                         f"{row['avg_nnz_per_row']:>9} {row['coarsening_ratio']:>7}")
        return "\n".join(lines) + "\n"
    raise AmgError(f"unknown report format {fmt!r} (text, json, csv)")


def main(argv=None):
    """``solve --cache DIR [--method pcg|bicgstab] [--rtol R] [--max-iters N] [--format F] [--history CSV]``."""
    import argparse
    import sys

    from . import hiercache, problems

    ap = argparse.ArgumentParser(prog="python -m paper_2102_07417_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sp = sub.add_parser("solve", help="solve A x = b on the GPU with a frozen reference hierarchy")
    sp.add_argument("--cache", required=True, help="hierarchy directory written by tools/export_hierarchy.py")
    sp.add_argument("--method", default="pcg")
    sp.add_argument("--rtol", type=float, default=1e-8)
    sp.add_argument("--max-iters", type=int, default=5000)
    sp.add_argument("--format", default="text", choices=("text", "json", "csv"))
    sp.add_argument("--history", help="write the residual history CSV here")
    sp.add_argument("--device", type=int, default=0)
    sp.add_argument("--devices", help="comma-separated GPU ids: partition the solve over them (one process)")
    args = ap.parse_args(argv)
    try:
        h = hiercache.load_hierarchy(args.cache)
        gen = h.meta.get("generator")
        b = problems.build_rhs(gen, h.levels[0].a.nrows) if gen else np.random.default_rng(42).standard_normal(
            h.levels[0].a.nrows)
        _, report, _ = run_solve(h.levels[0].a, b, {"solver.method": args.method, "solver.rtol": args.rtol,
                                                     "solver.max_iters": args.max_iters},
                                 hierarchy=h, device=args.device,
                                 devices=[int(d) for d in args.devices.split(",")] if args.devices else None)
    except (AmgError, OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    sys.stdout.write(report_emit(report, args.format))
    if args.history:
        with open(args.history, "w", encoding="ascii") as fh:
            fh.write("iteration,relative_residual\n")
            for it, res in report.history:
                fh.write(f"{it},{res!r}\n")
    return 0 if report.converged else 2
