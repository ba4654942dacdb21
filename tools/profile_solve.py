"""One device PCG solve for profiling (ncu launch lists / full captures).

    python tools/profile_solve.py --config c1_poisson7_64 [--graph 0|1|2] [--solves 1]
                                  [--spmv-only] [--opt key=value ...]

--graph 0 launches every kernel eagerly (each launch visible to ncu);
the kernels and their order are the same as inside the while-loop graph.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1_poisson7_64")
    ap.add_argument("--graph", type=int, default=0)
    ap.add_argument("--solves", type=int, default=1)
    ap.add_argument("--spmv-only", action="store_true")
    ap.add_argument("--levels", action="store_true", help="time every level's SpMVs and the coarse solve")
    ap.add_argument("--opt", action="append", default=[])
    args = ap.parse_args()
    import numpy as np

    import paper_2102_07417_b200 as amg
    from paper_2102_07417_b200 import hiercache, problems

    h = hiercache.load_hierarchy(os.path.join(ROOT, "hier_cache", args.config))
    opts = dict(kv.split("=") for kv in args.opt)
    dh = amg.DeviceHierarchy.from_reference(h, options={k: int(v) for k, v in opts.items()})
    dh.set_option("graph", args.graph)
    if args.spmv_only:
        for slot in ("a", "g", "gt", "p", "pt"):
            print(slot, dh.time_spmv(0, slot, reps=5))
        return
    if args.levels:
        for k, lv in enumerate(h.levels):
            slots = ("a", "g", "gt", "p", "pt") if lv.p is not None else ("a",)
            def t(k, s):
                try:
                    return f"{1e3 * dh.time_spmv(k, s, reps=20):.1f}us"
                except Exception as exc:  # levels folded into the tail kernel
                    return f"n/a({type(exc).__name__})"
            print(f"L{k} n={lv.a.nrows} nnz={lv.a.nnz} " + " ".join(f"{s}={t(k, s)}" for s in slots))
        print(f"coarse {t(-1, 'a')}")
    b = problems.build_rhs(args.config, h.levels[0].a.nrows)
    for _ in range(args.solves):
        t = time.perf_counter()
        r = amg.pcg(dh.A0, b, apply_m=dh.vcycle, config=amg.KrylovConfig(rtol=1e-8))
        print(f"its {r.n_iterations} relres {r.relres:.3e} solve_ms {r.solve_ms:.3f} wall {1e3*(time.perf_counter()-t):.1f}"
              f" stats {dh.stats()}")


if __name__ == "__main__":
    main()
