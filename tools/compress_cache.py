"""Re-save every hier_cache array file compressed (np.savez_compressed / npy -> npz untouched)."""
import glob
import os
import sys

import numpy as np

root = sys.argv[1] if len(sys.argv) > 1 else "hier_cache"
for f in sorted(glob.glob(os.path.join(root, "*", "*.npz"))):
    with np.load(f) as z:
        d = {k: z[k] for k in z.files}
    before = os.path.getsize(f)
    np.savez_compressed(f, **d)
    print(f, before >> 20, "->", os.path.getsize(f) >> 20, "MiB")
