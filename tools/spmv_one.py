"""Time (and let ncu capture) the SpMV of one matrix of a frozen hierarchy.

    python tools/spmv_one.py CONFIG LEVEL SLOT [--opt k=v ...] [--reps N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("level", type=int)
ap.add_argument("slot")
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
import paper_2102_07417_b200 as amg  # noqa: E402
from paper_2102_07417_b200 import hiercache  # noqa: E402

h = hiercache.load_hierarchy(os.path.join(ROOT, "hier_cache", a.config))
opts = {k: int(v) for k, v in (o.split("=") for o in a.opt)}
dh = amg.DeviceHierarchy.from_reference(h, options=opts or None)
ms = dh.time_spmv(a.level, a.slot, reps=a.reps)
st, ve = dh.matrix_bytes(a.level, a.slot)
print(f"{a.config} L{a.level}.{a.slot} {dh.layout(a.level, a.slot)} {opts}: {ms * 1e3:.2f} us, "
      f"{(st + ve) / (ms * 1e-3) / 1e9:.0f} GB/s over {st + ve} layout bytes")
