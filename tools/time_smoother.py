"""Device time of one FSAI smoother step from zero (x = w G^T G b) per level,
fused (fsai_fused) vs the two-kernel path.

    python tools/time_smoother.py c2_hetero27_128 [--levels 2] [--opt k=v ...]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--opt", action="append", default=[])
    args = ap.parse_args()
    import paper_2102_07417_b200 as amg
    from paper_2102_07417_b200 import hiercache

    h = hiercache.load_hierarchy(os.path.join(ROOT, "hier_cache", args.config))
    extra = {k: int(v) for k, v in (kv.split("=") for kv in args.opt)}
    for fused in (1, 0):
        dh = amg.DeviceHierarchy.from_reference(h, options={"fused": fused, **extra})
        st = dh.stats()
        for k in range(min(args.levels, h.n_levels - 1)):
            ms = dh.time_spmv(k, "smooth", reps=args.reps)
            print(json.dumps({"config": args.config, "level": k, "fused_opt": fused, "opts": extra,
                              "fused_here": bool((st["fused_levels"] >> k) & 1), "us": round(ms * 1e3, 2)}), flush=True)
        dh.close()


if __name__ == "__main__":
    main()
