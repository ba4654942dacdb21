"""Re-save a frozen hierarchy in another storage mode (e.g. compact -> lean).

    python tools/convert_cache.py hier_cache/c1_poisson7_64 [--mode lean] [--out DIR]

Loads with full digest verification, writes the new mode next to it (or in
place), and verifies the rewritten cache rebuilds bit for bit (digests).
"""
import argparse
import os
import shutil
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_07417_b200 import hiercache  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--mode", default="lean")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t0 = time.time()
    h = hiercache.load_hierarchy(a.src, verify=True)
    man = h.meta
    flags = [lv.get("symmetrize_next", True) for lv in man["levels"]]
    out = a.out or a.src
    tmp = tempfile.mkdtemp(prefix="hier_", dir=os.path.dirname(os.path.abspath(out)))
    hiercache.save_hierarchy(h, tmp, mode=a.mode, generator=man["generator"], symmetrize_flags=flags,
                             extra=man.get("extra"))
    t1 = time.time()
    hiercache.load_hierarchy(tmp, verify=True)
    t2 = time.time()
    if os.path.exists(out):
        shutil.rmtree(out)
    os.rename(tmp, out)
    size = sum(os.path.getsize(os.path.join(out, f)) for f in os.listdir(out))
    print(f"{out}: mode {a.mode}, {size / 2**20:.1f} MiB, save {t1 - t0:.1f} s, verified reload {t2 - t1:.1f} s")


if __name__ == "__main__":
    main()
