"""Per-op timing of the cluster tail (AMGB200_TRACE=1): python tools/trace_tail.py CONFIG [key=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2102_07417_b200 as amg
from paper_2102_07417_b200 import hiercache

cfg = sys.argv[1]
opts = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
h = hiercache.load_hierarchy(os.path.join("hier_cache", cfg))
dh = amg.DeviceHierarchy.from_reference(h, options=opts)
y = np.random.default_rng(0).standard_normal(h.levels[0].a.nrows)
for _ in range(4):
    dh.vcycle(y)
print(cfg, opts, "tail_level", dh.stats()["tail_level"], flush=True)
