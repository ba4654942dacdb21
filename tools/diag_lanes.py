import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2102_07417_b200 as amg
from golden_io import load_spmv_case, load_case
m, x, y = load_spmv_case("spmv_ragged")
lens = np.diff(m.row_offsets)
for lanes in (1, 2, 4, 8):
    dh = amg.DeviceHierarchy.from_matrices([m], options={"lanes": lanes})
    got = dh.matrix(0, "a")(x)
    bad = np.flatnonzero(got != y)
    print(lanes, "bad rows", bad.size, "lengths", sorted(set(lens[bad].tolist()))[:40])
    dh.close()
