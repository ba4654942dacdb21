import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2102_07417_b200 as amg
from paper_2102_07417_b200 import hiercache
for cfg in sys.argv[1:]:
    h = hiercache.load_hierarchy('hier_cache/' + cfg)
    dh = amg.DeviceHierarchy.from_reference(h)
    y = np.random.default_rng(0).standard_normal(h.levels[0].a.nrows)
    import pynvml, torch
    pynvml.nvmlInit(); hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    a = torch.randn(4096, 4096, device='cuda')
    for _ in range(200): a @ a   # warm the clocks
    for _ in range(3): dh.vcycle(y)
    print('sm clock MHz', pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM), file=sys.stderr)
    print(cfg, dh.stats(), flush=True)
