"""Loaders for the committed golden fixtures (made by tools/make_golden.py
from the reference itself; nothing here touches /root/reference)."""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2102_07417_b200 import hiercache
from paper_2102_07417_b200.problems import Csr

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

HIER_CASES = [
    "poisson7_12_bicg",
    "poisson7_12",
    "hetero27_10",
    "rtanis7_12",
    "poisson2d_16_jacobi",
    "poisson1d_8_twogrid_jacobi",
    "poisson1d_8_twogrid_nu20",
    "poisson1d_8_twogrid_fsai",
    "poisson1d_50_single",
    "elasticity_3_bamg",
    "poisson2d_12_lu",
]
SPMV_CASES = ["spmv_ragged", "spmv_longrow", "spmv_random_spd"]


def cases_with(key):
    """Hierarchy cases whose reference record includes `key` ("pcg" / "bicgstab")."""
    out = []
    for n in HIER_CASES:
        with open(os.path.join(GOLDEN, n, "expect.json")) as f:
            if key in json.load(f):
                out.append(n)
    return out


def load_case(name):
    d = os.path.join(GOLDEN, name)
    h = hiercache.load_hierarchy(os.path.join(d, "hier"), verify=True)
    with np.load(os.path.join(d, "vectors.npz")) as z:
        vec = {k: z[k] for k in z.files}
    with open(os.path.join(d, "expect.json")) as f:
        exp = json.load(f)
    out = {"h": h, "vec": vec, "expect": exp, "y": vec["y"], "b": vec["b"]}
    return out


def load_spmv_case(name):
    with np.load(os.path.join(GOLDEN, name, "spmv.npz")) as z:
        nr, nc = (int(v) for v in z["shape"])
        m = Csr(nr, nc, z["row_offsets"], z["col_indices"], z["values"])
        return m, z["x"].copy(), z["y"].copy()


def matrices_of(h):
    """(level, slot, matrix) for every matrix of a hierarchy."""
    for k, lvl in enumerate(h.levels):
        yield k, "a", lvl.a
        if lvl.p is not None:
            yield k, "p", lvl.p
            yield k, "pt", lvl.pt
        sm = lvl.smoother
        if sm is not None and sm.kind == "fsai":
            yield k, "g", sm.gmat
            yield k, "gt", sm.gmat_t
