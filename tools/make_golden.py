"""Generate the committed golden fixtures under tests/golden/ from the REFERENCE.

Run in the build container only (imports amgkit from /root/reference):

    python tools/make_golden.py

For each case: the reference hierarchy (``amgkit.setup``) frozen in full
mode, seeded input vectors, and the reference's own outputs of every
hot-path function -- ``spmv`` of every matrix, ``apply_smoother``,
``coarse_solve``, ``vcycle`` and ``pcg`` (x, iterations, relres, history).
Extra ``spmv_*`` cases pin the row-sum order on rows of length 0..400.
"""
from __future__ import annotations

import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

from amgkit import (  # noqa: E402
    AmgConfig, KrylovConfig, SparseMatrix, apply_smoother, bicgstab, pcg, setup, spmv, vcycle,
)
from amgkit.problems import gen_elasticity3d, gen_poisson7  # noqa: E402
from conftest import poisson1d, poisson2d, random_spd  # noqa: E402  (reference fixtures)

from paper_2102_07417_b200 import hiercache, problems  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def _sm(m):
    return SparseMatrix(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values, check=True)


def hierarchy_case(name, A, cfg, seed=7, rtol=1e-8, max_iters=500, solve=True, bicg=False):
    d = os.path.join(OUT, name)
    if os.path.exists(d):
        shutil.rmtree(d)
    h = setup(A, cfg)
    hiercache.save_hierarchy(h, os.path.join(d, "hier"), mode="full")
    rng = np.random.default_rng(seed)
    n = A.nrows
    vec = {}
    exp = {"n_levels": h.n_levels, "factor_kind": h.factor_kind, "sizes": [l.a.nrows for l in h.levels]}
    for k, lvl in enumerate(h.levels):
        mats = {"a": lvl.a}
        if lvl.p is not None:
            mats.update(p=lvl.p, pt=lvl.pt)
        if lvl.smoother is not None and lvl.smoother.kind == "fsai":
            mats.update(g=lvl.smoother.gmat, gt=lvl.smoother.gmat_t)
        for slot, m in mats.items():
            x = rng.uniform(-1, 1, m.ncols)
            vec[f"spmv_L{k}_{slot}_x"] = x
            vec[f"spmv_L{k}_{slot}_y"] = spmv(m, x)
        if lvl.smoother is not None:
            b = rng.uniform(-1, 1, lvl.a.nrows)
            x0 = rng.uniform(-1, 1, lvl.a.nrows)
            vec[f"smooth_L{k}_b"] = b
            vec[f"smooth_L{k}_x0"] = x0
            for steps in (1, 2):
                vec[f"smooth_L{k}_zero_{steps}"] = apply_smoother(lvl.smoother, lvl.a, b, np.zeros_like(b), steps)
                vec[f"smooth_L{k}_x0_{steps}"] = apply_smoother(lvl.smoother, lvl.a, b, x0, steps)
    yc = rng.uniform(-1, 1, h.levels[-1].a.nrows)
    vec["coarse_y"] = yc
    vec["coarse_z"] = h.coarse_solve(yc)
    y = rng.uniform(-1, 1, n)
    vec["y"] = y
    vec["vcycle_z"] = vcycle(h, y)
    b = np.random.default_rng(42).uniform(-1, 1, n)
    vec["b"] = b
    if solve:
        res = pcg(lambda v: spmv(A, v), b, apply_m=lambda r: vcycle(h, r),
                  config=KrylovConfig(rtol=rtol, max_iters=max_iters, record_history=True))
        vec["pcg_x"] = res.x
        exp["pcg"] = {"rtol": rtol, "max_iters": max_iters, "converged": bool(res.converged),
                      "n_iterations": int(res.n_iterations), "relres": float(res.relres),
                      "history": [float(r) for _, r in res.history]}
    if bicg:
        res = bicgstab(lambda v: spmv(A, v), b, apply_m=lambda r: vcycle(h, r),
                       config=KrylovConfig(rtol=rtol, max_iters=max_iters, record_history=True))
        vec["bicgstab_x"] = res.x
        exp["bicgstab"] = {"rtol": rtol, "max_iters": max_iters, "converged": bool(res.converged),
                           "n_iterations": int(res.n_iterations), "relres": float(res.relres),
                           "restarts": int(res.restarts), "history": [float(r) for _, r in res.history]}
    np.savez(os.path.join(d, "vectors.npz"), **vec)
    with open(os.path.join(d, "expect.json"), "w") as f:
        json.dump(exp, f, indent=1)
    print(name, exp["sizes"], exp.get("pcg", {}).get("n_iterations"))


def spmv_case(name, A, seed=11):
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(A.ncols) * 10.0 ** rng.integers(-3, 3, A.ncols)
    np.savez(os.path.join(d, "spmv.npz"), shape=np.asarray(A.shape), row_offsets=A.row_offsets,
             col_indices=A.col_indices, values=A.values, x=x, y=spmv(A, x))
    print(name, A.shape, A.nnz)


def ragged_matrix(rng, lengths, ncols):
    rows, cols = [], []
    for i, L in enumerate(lengths):
        c = np.sort(rng.choice(ncols, size=L, replace=False))
        rows.append(np.full(L, i))
        cols.append(c)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = rng.standard_normal(r.size) * 10.0 ** rng.integers(-4, 4, r.size)
    m = sp.csr_matrix((v, (r, c)), shape=(len(lengths), ncols))
    m.sort_indices()
    return SparseMatrix.from_scipy(m)


def main():
    os.makedirs(OUT, exist_ok=True)
    # scalar Poisson, FSAI (config-1 recipe at 12^3)
    hierarchy_case("poisson7_12", gen_poisson7(12, 12, 12), AmgConfig(smoother="fsai"))
    # 27-point heterogeneous diffusion (config-2 generator at 10^3)
    hierarchy_case("hetero27_10", _sm(problems.hetero27(10, 10, 10, sigma=2.0, seed=42)),
                   AmgConfig(smoother="fsai", max_coarse=60))
    # anisotropic 7-point (config-4 generator at 12^3)
    hierarchy_case("rtanis7_12", _sm(problems.rtanis7(12, 12, 12, 1.0, 1.0, 1e-3)),
                   AmgConfig(smoother="fsai", max_coarse=50))
    # Jacobi hierarchy of test_krylov.py:138-147 / test_hierarchy.py
    hierarchy_case("poisson2d_16_jacobi", poisson2d(16), AmgConfig(max_coarse=40))
    # two-grid fixtures of test_hierarchy.py:86-117
    hierarchy_case("poisson1d_8_twogrid_jacobi", poisson1d(8), AmgConfig(max_coarse=4, max_levels=2), solve=False)
    hierarchy_case("poisson1d_8_twogrid_nu20", poisson1d(8), AmgConfig(max_coarse=4, max_levels=2, nu1=2, nu2=0),
                   solve=False)
    hierarchy_case("poisson1d_8_twogrid_fsai", poisson1d(8), AmgConfig(max_coarse=4, max_levels=2, smoother="fsai"),
                   solve=False)
    # single level = direct solve (test_hierarchy.py:32-40)
    hierarchy_case("poisson1d_50_single", poisson1d(50), AmgConfig(max_coarse=200))
    # elasticity with BAMG + rigid body modes (config-3 recipe at 3^3 elements)
    a, coords = gen_elasticity3d(3, 3, 3)
    hierarchy_case("elasticity_3_bamg", a, AmgConfig(smoother="fsai", interp="bamg", testspace="rigid_body",
                                                      n_test_vectors=6, coords=coords, max_coarse=50))
    # nonsymmetric coarse operators -> LU coarsest factor (hierarchy.py:143-147)
    hierarchy_case("poisson2d_12_lu", poisson2d(12),
                   AmgConfig(max_coarse=30, filter_target="operator", filter_rho=0.6), solve=False, bicg=True)
    hierarchy_case("poisson7_12_bicg", gen_poisson7(12, 12, 12), AmgConfig(smoother="fsai"), solve=False, bicg=True)
    # row-sum order: ragged rows incl. empty and > 128 entries (recursive pairwise)
    rng = np.random.default_rng(5)
    lengths = np.concatenate([np.arange(0, 140), [0, 0, 200, 257, 300, 400, 129, 130, 136, 137],
                              rng.integers(0, 40, 200)])
    spmv_case("spmv_ragged", ragged_matrix(rng, lengths, 600))
    # one row longer than a staging tile (2048 entries) + short rows
    spmv_case("spmv_longrow", ragged_matrix(rng, [3, 2500, 0, 7, 5000, 1], 6000))
    spmv_case("spmv_random_spd", random_spd(np.random.default_rng(2024), 300, density=0.05))


if __name__ == "__main__":
    main()
