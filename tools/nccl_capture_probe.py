"""Which multi-GPU NCCL calls capture into the conditional WHILE body? (one GPU, one-rank comm)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2102_07417_b200 as amg  # noqa: E402
from golden_io import load_case  # noqa: E402

c = load_case("poisson7_12")
base = {"overlap_test": 1, "small_rows_per_sm": 1, "dict": 0}
d0 = amg.DeviceHierarchy.from_reference(c["h"], options=base)
r0 = amg.pcg(d0.A0, c["b"], apply_m=d0.vcycle, config=amg.KrylovConfig(rtol=1e-10))
for mode, what in ((2, "dot all-gathers"), (3, "p2p on the comm stream (fork/join)"), (1, "both"),
                   (4, "p2p on the main stream"), (5, "fork/join with a plain kernel on the comm stream")):
    d = amg.DeviceHierarchy.from_reference(c["h"], options={**base, "nccl_selftest": mode})
    r = amg.pcg(d.A0, c["b"], apply_m=d.vcycle, config=amg.KrylovConfig(rtol=1e-10))
    print(f"nccl_selftest={mode} ({what}): graph_mode {d.stats()['graph_mode']}, its {r.n_iterations} "
          f"(vs {r0.n_iterations}), x bit-identical {np.array_equal(r.x, r0.x)}", flush=True)
    d.close()
