"""Per-call wall time of the public pcg() with pinned host vectors vs its device time (e2e overheads)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2102_07417_b200 as amg
from paper_2102_07417_b200 import hiercache, problems
h = hiercache.load_hierarchy('hier_cache/c2_hetero27_128', verify=False)
dh = amg.DeviceHierarchy.from_reference(h)
b = problems.build_rhs('c2_hetero27_128', h.levels[0].a.nrows)
cfg = amg.KrylovConfig(rtol=1e-8, max_iters=5000)
b_pin = torch.from_numpy(b).pin_memory()
amg.pcg(dh.A0, b_pin, apply_m=dh.vcycle, config=cfg)
for i in range(10):
    t0 = time.perf_counter(); r = amg.pcg(dh.A0, b_pin, apply_m=dh.vcycle, config=cfg); t1 = time.perf_counter()
    print(f"call {i}: wall {1e3*(t1-t0):.3f} ms  device {r.solve_ms:.3f} ms  its {r.n_iterations}", flush=True)
