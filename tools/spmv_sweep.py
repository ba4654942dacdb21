"""Per-matrix SpMV timing (CUDA events, back-to-back launches) and achieved GB/s.

    python tools/spmv_sweep.py CONFIG [--opt key=value ...] [--levels 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    import paper_2102_07417_b200 as amg
    from paper_2102_07417_b200 import hiercache

    h = hiercache.load_hierarchy(os.path.join(ROOT, "hier_cache", args.config))
    opts = {k: int(v) for k, v in (kv.split("=") for kv in args.opt)}
    dh = amg.DeviceHierarchy.from_reference(h, options=opts)
    print(args.config, opts, dh.stats()["tail_level"])
    for k, lv in enumerate(h.levels[: args.levels]):
        mats = {"a": lv.a}
        if lv.p is not None:
            mats.update(p=lv.p, pt=lv.pt, g=lv.smoother.gmat, gt=lv.smoother.gmat_t)
        for slot, m in mats.items():
            ms = dh.time_spmv(k, slot, reps=args.reps)
            byts = 12 * m.nnz + 4 * (m.nrows + 1) + 8 * m.ncols + 8 * m.nrows
            print(f"L{k}.{slot:2s} rows {m.nrows:9d} nnz {m.nnz:10d} ({m.nnz/max(m.nrows,1):5.1f}/row) "
                  f"{ms*1e3:8.2f} us  {byts/ms/1e6:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
