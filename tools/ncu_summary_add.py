"""Add one kernel capture to profiles/ncu_summary.json.

    python tools/ncu_summary_add.py CONFIG MATRIX LAYOUT REPORT.ncu-rep "kernel description" profiles/SOURCE.txt

Reads dram bytes and duration of the (single) captured launch from the report (ncu --page raw --csv)
and records them under CONFIG, keyed by the matrix (e.g. L1.a) and device layout the capture ran on.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg, matrix, layout, rep, desc, src = sys.argv[1:7]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, val = rows[0], rows[1], rows[-1]


def get(name):
    i = hdr.index(name)
    v, u = float(val[i]), units[i]
    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3}.get(u, 1.0)
    return v * scale


p = os.path.join(ROOT, "profiles", "ncu_summary.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d[cfg] = {
    "kernel": desc, "matrix": matrix, "layout": layout,
    "dram_bytes_per_launch": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
    "ncu_duration_us": get("gpu__time_duration.sum"),
    "source": src,
}
json.dump(d, open(p, "w"), indent=1)
print(json.dumps(d[cfg], indent=1))
