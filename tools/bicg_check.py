import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2102_07417_b200 as amg
from golden_io import load_case
from oracle import solve as O
for name in ("poisson2d_12_lu", "poisson7_12_bicg"):
    c = load_case(name); exp = c["expect"]["bicgstab"]
    dh = amg.DeviceHierarchy.from_reference(c["h"])
    r = amg.bicgstab(dh.A0, c["b"], apply_m=dh.vcycle, config=amg.KrylovConfig(rtol=1e-8, max_iters=500, record_history=True))
    true = np.linalg.norm(c["b"] - O.spmv(c["h"].levels[0].a, r.x)) / np.linalg.norm(c["b"])
    print(name, "device its", r.n_iterations, "ref its", exp["n_iterations"], "relres", r.relres, "true", true, "restarts", r.restarts, exp["restarts"])
    print("  dev", [f"{v:.3e}" for _, v in r.history[:12]])
    print("  ref", [f"{v:.3e}" for v in exp["history"][:12]])
    zd = dh.vcycle(c["y"]); zr = c["vec"]["vcycle_z"]
    print("  vcycle relerr", np.abs(zd - zr).max() / max(1, np.abs(zr).max()))
