"""Time the fine-grid operator A_0 of a config alone (no hierarchy needed) on
every applicable device layout: CUDA events around back-to-back launches.

    python tools/time_a0.py c2_hetero27_128 [--reps 50]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--only", type=int, default=None, help="symm option to run (default both)")
    ap.add_argument("--opt", action="append", default=[], help="extra key=value handle options")
    args = ap.parse_args()
    import numpy as np

    import paper_2102_07417_b200 as amg
    from paper_2102_07417_b200 import problems
    from oracle import solve as O

    for cfg in args.configs:
        m = problems.build_config(cfg)
        x = np.random.default_rng(1).uniform(-1, 1, m.ncols)
        want = None
        extra = {k: int(v) for k, v in (kv.split("=") for kv in args.opt)}
        for opts in ({"symm": 1}, {"symm": 0}):
            if args.only is not None and opts["symm"] != args.only:
                continue
            opts = {**opts, **extra}
            dh = amg.DeviceHierarchy.from_matrices([m], options=opts)
            ms = dh.time_spmv(0, "a", reps=args.reps)
            got = dh.matrix(0, "a")(x)
            if want is None and m.nrows <= 3_000_000 and not args.no_check:
                want = O.spmv(m, x)
            exact = None if want is None else bool(np.array_equal(got, want))
            model = 12 * m.nnz + 4 * (m.nrows + 1) + 8 * m.ncols + 8 * m.nrows
            print(json.dumps({"config": cfg, "opts": opts, "layout": dh.layout(0, "a"), "rows": m.nrows, "nnz": m.nnz,
                              "us": round(ms * 1e3, 2), "model_gbs": round(model / ms / 1e6),
                              "bit_exact_vs_oracle": exact}), flush=True)
            dh.close()


if __name__ == "__main__":
    main()
