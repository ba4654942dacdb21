"""V-cycle / PCG with tail variants vs the default: bitwise V-cycle equality, iterations, time.

    python tools/tail_check.py CONFIG "k=v k=v" ["k=v" ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2102_07417_b200 as amg  # noqa: E402
from paper_2102_07417_b200 import hiercache, problems  # noqa: E402

cfg = sys.argv[1]
h = hiercache.load_hierarchy(os.path.join(ROOT, "hier_cache", cfg))
b = problems.build_rhs(cfg, h.levels[0].a.nrows)
y = np.random.default_rng(0).uniform(-1, 1, h.levels[0].a.nrows)
ref = amg.DeviceHierarchy.from_reference(h)
z0 = ref.vcycle(y)
r0 = amg.pcg(ref.A0, b, apply_m=ref.vcycle, config=amg.KrylovConfig(rtol=1e-8))
print(f"default: tail_level {ref.stats()['tail_level']}, {r0.n_iterations} its, {r0.solve_ms / r0.n_iterations:.4f} ms/it")
for spec in sys.argv[2:]:
    opts = {k: int(v) for k, v in (t.split("=") for t in spec.split())}
    d = amg.DeviceHierarchy.from_reference(h, options=opts)
    z = d.vcycle(y)
    ms = []
    for _ in range(3):
        r = amg.pcg(d.A0, b, apply_m=d.vcycle, config=amg.KrylovConfig(rtol=1e-8))
        ms.append(r.solve_ms / r.n_iterations)
    st = d.stats()
    print(f"{spec}: tail_level {st['tail_level']} ctas {st['cluster']} graph {st['graph_mode']}, vcycle bitwise "
          f"{np.array_equal(z, z0)} (max diff {np.abs(z - z0).max():.2e}), {r.n_iterations} its, "
          f"{min(ms):.4f} ms/it", flush=True)
    d.close()
