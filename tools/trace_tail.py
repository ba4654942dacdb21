import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2102_07417_b200 as amg
from paper_2102_07417_b200 import hiercache
for cfg in sys.argv[1:]:
    h = hiercache.load_hierarchy('hier_cache/' + cfg)
    dh = amg.DeviceHierarchy.from_reference(h)
    y = np.random.default_rng(0).standard_normal(h.levels[0].a.nrows)
    for _ in range(3): dh.vcycle(y)
    print(cfg, dh.stats(), flush=True)
