import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2102_07417_b200 as amg
from paper_2102_07417_b200 import hiercache, problems
h = hiercache.load_hierarchy('hier_cache/c2_hetero27_128', verify=False)
dh = amg.DeviceHierarchy.from_reference(h)
b = problems.build_rhs('c2_hetero27_128', h.levels[0].a.nrows)
cfg = amg.KrylovConfig(rtol=1e-8)
b_pin = torch.from_numpy(b).pin_memory()
b_dev = torch.from_numpy(b).cuda()
for name, bb in (("pinned", b_pin), ("device", b_dev), ("numpy", b)):
    amg.pcg(dh.A0, bb, apply_m=dh.vcycle, config=cfg)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = amg.pcg(dh.A0, bb, apply_m=dh.vcycle, config=cfg); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, "wall ms", np.median(ts) * 1e3, "solve_ms", r.solve_ms, "its", r.n_iterations, "stats e2e", dh.stats()["e2e_ms"])
