"""Run the REFERENCE hierarchy setup once and freeze it (build container only).

Usage: python tools/export_hierarchy.py <config> [--out hier_cache] [--mode lean|compact|full]
                                        [--solve] [--state DIR] [--oneshot]

Imports ``amgkit`` from /root/reference/pkg/src (it is not available on the
GPU box), builds A_0 with the config's generator, runs the reference setup
(``amgkit/hierarchy.py:155-223``) level by level through
``tools/setup_resumable.py`` (every finished level is pickled under --state,
so an interrupted multi-hour setup resumes where it stopped; ``--oneshot``
calls ``amgkit.setup`` directly instead), and writes the result with
:func:`paper_2102_07417_b200.hiercache.save_hierarchy` (lean by default:
G's pattern only, see hiercache.py).
With ``--solve`` it also runs the reference solve
``pcg(spmv(A0,.), b, vcycle(h,.), KrylovConfig(rtol=1e-8, record_history=True))``
on ``b = default_rng(42).uniform(-1, 1, n)`` and records iterations, final
relres and the residual history in the manifest (the iteration-count parity
record for the device solve).
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import amgkit  # noqa: E402
from amgkit import AmgConfig, KrylovConfig, SparseMatrix, is_symmetric, pcg, setup, spmv, vcycle  # noqa: E402

from paper_2102_07417_b200 import hiercache, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "hier_cache"))
    ap.add_argument("--mode", default="lean", choices=("lean", "compact", "full"))
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--state", default=None, help="per-level setup state (default <out>/.setup_<config>)")
    ap.add_argument("--oneshot", action="store_true", help="amgkit.setup in one call (no per-level state)")
    args = ap.parse_args()

    fn, gargs, gkw, recipe = problems.CONFIGS[args.config]
    a0, coords = problems.build_config(args.config, with_coords=True)
    A = SparseMatrix(a0.nrows, a0.ncols, a0.row_offsets, a0.col_indices, a0.values, check=True)
    cfg = dict(recipe)
    if coords is not None:
        cfg["coords"] = coords
    t0 = time.perf_counter()
    if args.oneshot:
        h = setup(A, AmgConfig(**cfg))
    else:
        from setup_resumable import setup_resumable

        state = args.state or os.path.join(args.out, f".setup_{args.config}")
        h = setup_resumable(A, AmgConfig(**cfg), state, log=lambda m: print(m, flush=True))
    t_setup = time.perf_counter() - t0
    flags = []
    for lvl in h.levels[:-1]:
        flags.append(bool(is_symmetric(lvl.a)) if h.symmetric else False)
    extra = {
        "recipe": {k: v for k, v in recipe.items()},
        "setup_seconds": t_setup,
        "peak_rss_mb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024.0,
        "amgkit_version": amgkit.__version__,
        "numpy": np.__version__,
        "omegas": [float(l.smoother.omega) for l in h.levels if l.smoother is not None],
        "sizes": [int(l.a.nrows) for l in h.levels],
        "nnz": [int(l.a.nnz) for l in h.levels],
    }
    if args.solve:
        b = problems.build_rhs(args.config, A.nrows)
        t1 = time.perf_counter()
        res = pcg(lambda v: spmv(A, v), b, apply_m=lambda r: vcycle(h, r),
                  config=KrylovConfig(rtol=1e-8, record_history=True))
        t2 = time.perf_counter()
        extra["reference_solve"] = {
            "rhs": "uniform(-1,1) seed 42",
            "converged": bool(res.converged),
            "n_iterations": int(res.n_iterations),
            "relres": float(res.relres),
            "history": [float(r) for _, r in res.history],
            "solve_seconds": t2 - t1,
            "ms_per_iter": 1e3 * (t2 - t1) / max(res.n_iterations, 1),
        }
    out = os.path.join(args.out, args.config)
    man = hiercache.save_hierarchy(h, out, mode=args.mode, generator=args.config,
                                   symmetrize_flags=flags, extra=extra)
    # verify the compact form rebuilds bit-identically before declaring success
    hiercache.load_hierarchy(out, verify=True)
    print(json.dumps({k: man["extra"][k] for k in ("setup_seconds", "sizes", "omegas")}))
    if "reference_solve" in extra:
        rs = extra["reference_solve"]
        print("reference solve:", rs["n_iterations"], rs["relres"], rs["ms_per_iter"])


if __name__ == "__main__":
    main()
