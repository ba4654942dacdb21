"""Print the device layout (and stored bytes) chosen for every matrix of a frozen hierarchy.

    python tools/layouts.py c2_hetero27_128 [c1_poisson7_64 ...] [--opt key=value ...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--time", action="store_true", help="also time every SpMV (CUDA events, 20 reps)")
    a = ap.parse_args()
    import paper_2102_07417_b200 as amg
    from paper_2102_07417_b200 import hiercache

    opts = {k: int(v) for k, v in (o.split("=") for o in a.opt)}
    for cfg in a.configs:
        t0 = time.time()
        h = hiercache.load_hierarchy(os.path.join(ROOT, "hier_cache", cfg))
        t1 = time.time()
        dh = amg.DeviceHierarchy.from_reference(h, options=opts or None)
        t2 = time.time()
        rows = []
        for k, lv in enumerate(h.levels):
            mats = {"a": lv.a}
            if lv.p is not None:
                mats.update(p=lv.p, pt=lv.pt)
                if lv.smoother is not None and lv.smoother.kind == "fsai":
                    mats.update(g=lv.smoother.gmat, gt=lv.smoother.gmat_t)
            for slot, m in mats.items():
                st, ve = dh.matrix_bytes(k, slot)
                r = {"level": k, "slot": slot, "rows": m.nrows, "nnz": m.nnz, "layout": dh.layout(k, slot),
                     "stored_mb": round(st / 1e6, 3), "csr_mb": round((12 * m.nnz + 4 * m.nrows) / 1e6, 3)}
                if a.time:
                    ms = dh.time_spmv(k, slot, reps=20)
                    r["us"] = round(ms * 1e3, 2)
                    r["gbs"] = round((st + ve) / (ms * 1e-3) / 1e9, 1)
                rows.append(r)
        print(json.dumps({"config": cfg, "load_s": round(t1 - t0, 1), "upload_s": round(t2 - t1, 1),
                          "stats": dh.stats(), "matrices": rows}))
        dh.close()


if __name__ == "__main__":
    main()
