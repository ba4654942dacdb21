"""Aggregate ncu source-page samples per CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep [top]
Prints the lines with the most warp-stall samples and their dominant stall reasons.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
cur = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (int(r[0]), r[1][:110])
    if cur is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    if r[0]:  # the source line's own row carries the aggregate
        s = agg.setdefault(cur, {"samples": 0, "stalls": {}})
        try:
            s["samples"] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            pass
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    s["stalls"][k] = s["stalls"].get(k, 0) + int(v or 0)
                except ValueError:
                    pass
tot = sum(v["samples"] for v in agg.values()) or 1
print(f"total samples {tot}")
for (ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(v["stalls"].items(), key=lambda kv: -kv[1])[:3]
    print(f"{v['samples']:7d} {100 * v['samples'] / tot:5.1f}%  L{ln:<5d} {src.strip()[:90]}  | " +
          ", ".join(f"{k[6:]}={n}" for k, n in st))
