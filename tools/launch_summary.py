"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel share."""
import collections
import csv
import sys


def load(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def main(path, per_iter=None):
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d["Kernel Name"].split("(")[0][:48] + " grid" + ("=1" if d["Grid Size"].startswith("(1,") else ">1")
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot/1e3:.1f} us total")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:6d} {v[1]/1e3:10.1f} us {100*v[1]/tot:5.1f}%  avg {v[1]/v[0]/1e3:7.2f} us  {k}")
    if per_iter:
        print("per iteration us:", tot / 1e3 / per_iter)


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
