import sys, os, ctypes
sys.path.insert(0, '/root/repo')
import paper_2102_07417_b200 as amg
from paper_2102_07417_b200 import hiercache, _capi as C
opts = {k: int(v) for k, v in (a.split('=') for a in sys.argv[1:] if '=' in a)}
for cfg in [a for a in sys.argv[1:] if '=' not in a]:
    h = hiercache.load_hierarchy('hier_cache/' + cfg)
    dh = amg.DeviceHierarchy.from_reference(h, options=opts)
    ms = C.D(0.0)
    C.check(C.lib().amg_time_spmv(dh._h, -1, 0, 20, ctypes.byref(ms)))
    print(cfg, opts, 'n_coarse', h.levels[-1].a.nrows, 'coarse solve us', ms.value * 1e3)
