"""Hierarchy cache: compact form rebuilds the reference's hierarchy bit for bit;
bench generators match the reference generators."""
import os

import numpy as np
import pytest

from conftest import have_reference
from golden_io import load_case
from paper_2102_07417_b200 import hiercache, problems


def _eq(a, b):
    return (a.nrows == b.nrows and a.ncols == b.ncols and np.array_equal(a.row_offsets, b.row_offsets)
            and np.array_equal(a.col_indices, b.col_indices) and np.array_equal(a.values, b.values))


def test_full_roundtrip(tmp_path):
    c = load_case("poisson7_12")
    h = c["h"]
    hiercache.save_hierarchy(h, str(tmp_path / "h"), mode="full")
    h2 = hiercache.load_hierarchy(str(tmp_path / "h"))
    for l1, l2 in zip(h.levels, h2.levels):
        assert _eq(l1.a, l2.a)
    np.testing.assert_array_equal(h.factor[0], h2.factor[0])


def test_compact_rebuild_matches_digests(tmp_path):
    # the rebuilt A_{k+1} = galerkin(A_k, P_k), P^T, G^T must equal what the reference stored
    c = load_case("poisson7_12")
    h = c["h"]
    a0 = problems.poisson7(12, 12, 12)
    assert _eq(a0, h.levels[0].a)
    for k in range(h.n_levels - 1):
        lv = h.levels[k]
        assert _eq(hiercache.galerkin_product(lv.a, lv.p, True), h.levels[k + 1].a)
        assert _eq(hiercache.transpose(lv.p), lv.pt)
        assert _eq(hiercache.transpose(lv.smoother.gmat), lv.smoother.gmat_t)


def test_digest_mismatch_is_loud(tmp_path):
    c = load_case("poisson7_12")
    d = str(tmp_path / "h")
    hiercache.save_hierarchy(c["h"], d, mode="full")
    z = dict(np.load(os.path.join(d, "L0_a.npz")))
    z["values"] = z["values"].copy()
    z["values"][0] += 1.0
    np.savez(os.path.join(d, "L0_a.npz"), **z)
    with pytest.raises(ValueError, match="digest"):
        hiercache.load_hierarchy(d)


@pytest.mark.skipif(not have_reference(), reason="reference package only in the build container")
def test_generators_match_reference():
    from amgkit.problems import gen_poisson7, gen_rotated_anisotropy
    from amgkit import SparseMatrix

    assert _eq(problems.poisson7(5, 6, 7), gen_poisson7(5, 6, 7))
    assert _eq(problems.rtanis7(6, 5, 7, 1.0, 1.0, 1e-3), gen_rotated_anisotropy(6, 5, 7, theta=0, kx=1, ky=1, kz=1e-3))
    a = problems.hetero27(6, 5, 7, sigma=2.0, seed=3)
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_offsets))
    b = SparseMatrix.from_coo(rows, a.col_indices, a.values, a.shape)
    assert _eq(a, b)
    assert a.nnz == (3 * 6 - 2) * (3 * 5 - 2) * (3 * 7 - 2)


def test_hetero27_sizes_and_symmetry():
    a = problems.hetero27(7, 6, 5, sigma=2.0, seed=1)
    assert a.nnz == 19 * 16 * 13
    rows = np.repeat(np.arange(a.nrows), np.diff(a.row_offsets))
    d = np.zeros((a.nrows, a.nrows))
    d[rows, a.col_indices] = a.values
    assert np.array_equal(d, d.T)
    assert np.linalg.eigvalsh(d).min() > 0
    blk = problems.conductivity(8, 8, 8, 3.0, 42, block=4)
    assert np.unique(blk).size == 8


def test_report_emit_matches_reference_schema():
    from paper_2102_07417_b200.solve import SolveReport, level_table, report_emit, complexities

    c = load_case("poisson7_12")
    h = c["h"]
    rep = SolveReport("pcg", True, 10, 1e-8, 3e-9, 1.2, 1.3, h.n_levels, level_table(h), 0.1, 0.2, 0.3,
                      h.levels[0].a.nrows, h.levels[0].a.nnz, [(0, 1.0)])
    doc = __import__("json").loads(report_emit(rep, "json"))
    assert doc["schema_version"] == 1 and doc["n_iterations"] == 10 and len(doc["levels"]) == h.n_levels
    assert report_emit(rep, "csv").startswith("level,n,nnz,avg_nnz_per_row,coarsening_ratio")
    if have_reference():
        from amgkit.cli import report_emit as ref_emit
        from amgkit.hierarchy import SolveReport as RefReport, level_table as ref_table

        assert level_table(h) == ref_table(h)
        ref = RefReport(**rep.__dict__)
        for fmt in ("json", "csv", "text"):
            assert report_emit(rep, fmt) == ref_emit(ref, fmt)


@pytest.mark.parametrize("case", ["poisson7_12", "hetero27_10", "rtanis7_12", "elasticity_3_bamg",
                                  "poisson1d_8_twogrid_fsai", "poisson2d_16_jacobi"])
def test_lean_cache_replays_fsai_bit_for_bit(tmp_path, case):
    # lean mode stores only G's pattern; the FSAI coefficients are replayed with
    # scipy's own LAPACK (csrc/fsai_host.c) and must equal the reference's G
    h = load_case(case)["h"]
    d = str(tmp_path / "lean")
    flags = [True] * h.n_levels
    hiercache.save_hierarchy(h, d, mode="lean", symmetrize_flags=flags)
    assert not any(f.endswith("_g.npz") for f in os.listdir(d))
    h2 = hiercache.load_hierarchy(d, verify=True, threads=3)
    for l1, l2 in zip(h.levels, h2.levels):
        assert _eq(l1.a, l2.a)
        if l1.smoother is not None and l1.smoother.kind == "fsai":
            assert _eq(l1.smoother.gmat, l2.smoother.gmat)
            assert _eq(l1.smoother.gmat_t, l2.smoother.gmat_t)
        if l1.p is not None:
            assert _eq(l1.p, l2.p)
            assert _eq(l1.pt, l2.pt)


def test_lean_replay_is_loud_on_a_wrong_pattern(tmp_path):
    h = load_case("poisson7_12")["h"]
    d = str(tmp_path / "lean")
    hiercache.save_hierarchy(h, d, mode="lean", symmetrize_flags=[True] * h.n_levels)
    z = dict(np.load(os.path.join(d, "L1_gpat.npz")))
    rel = z["rel"].copy()
    k = int(np.flatnonzero(rel > 1)[0])
    rel[k] -= 1  # move one off-diagonal entry of G_1 to a neighbouring column
    z["rel"] = rel
    np.savez_compressed(os.path.join(d, "L1_gpat.npz"), **z)
    with pytest.raises(ValueError, match="digest|FSAI replay"):
        hiercache.load_hierarchy(d)


def test_fsai_replay_matches_scipy_cho_solve():
    # the replay against scipy.linalg.cho_factor / cho_solve called as the
    # reference calls them (smoothers.py:84-91), on random SPD blocks
    import scipy.linalg as sla
    import scipy.sparse as sp
    from paper_2102_07417_b200.fsai_host import fsai_values
    from paper_2102_07417_b200.problems import Csr

    rng = np.random.default_rng(3)
    n = 60
    m = sp.random(n, n, density=0.3, random_state=4) + sp.eye(n) * 0.1
    a = (m @ m.T + sp.eye(n) * n).tocsr()
    a.sort_indices()
    A = Csr(n, n, a.indptr, a.indices, a.data)
    dense = a.toarray()
    offs, cols, want = [0], [], []
    for i in range(n):
        k = min(i, int(rng.integers(0, 9)))
        pat = np.sort(rng.choice(i, size=k, replace=False)) if k else np.zeros(0, dtype=np.int64)
        idx = np.concatenate([pat, [i]]).astype(np.int64)
        sub = dense[np.ix_(idx, idx)]
        c, low = sla.cho_factor(sub, lower=True, check_finite=False)
        e = np.zeros(idx.size)
        e[-1] = 1.0
        y = sla.cho_solve((c, low), e, check_finite=False)
        want.append(y / np.sqrt(y[-1]))
        cols.extend(idx.tolist())
        offs.append(len(cols))
    got = fsai_values(A, np.asarray(offs), np.asarray(cols), threads=4)
    np.testing.assert_array_equal(got, np.concatenate(want))


@pytest.mark.skipif(not have_reference(), reason="reference package only in the build container")
@pytest.mark.parametrize("n", [3, 6])
def test_elasticity3d_matches_reference_generator_at_sigma0(n):
    # config 3's generator (per-element lognormal E, unit cube h = 1/n) pinned to
    # the reference's gen_elasticity3d (problems.py:142-199): with sigma = 0 every
    # E is 1 and the Q1 stiffness scales with h in 3-D, so ours == h * reference
    # up to assembly-order rounding; same clamped-dof numbering, coords * h
    from amgkit.problems import gen_elasticity3d

    a, coords = problems.elasticity3d(n, n, n, sigma=0.0, nu=0.3, seed=7)
    r, rc = gen_elasticity3d(n, n, n, e=1.0, nu=0.3, bc="clamped")
    assert a.shape == r.shape == (3 * n * (n + 1) ** 2,) * 2
    np.testing.assert_array_equal(coords, np.asarray(rc) * (1.0 / n))

    def dense(m):
        d = np.zeros(m.shape)
        rows = np.repeat(np.arange(m.nrows), np.diff(m.row_offsets))
        np.add.at(d, (rows, m.col_indices), m.values)
        return d

    da, dr = dense(a), dense(r) / n
    scale = np.abs(dr).max()
    assert np.abs(da - dr).max() <= 1e-13 * scale
    # stored patterns agree except where exact cancellation leaves a rounding-level entry
    diff = (da != 0) ^ (dr != 0)
    assert np.all(np.abs(da[diff]) <= 1e-13 * scale) and np.all(np.abs(dr[diff]) <= 1e-13 * scale)


@pytest.mark.skipif(not have_reference(), reason="reference package only in the build container")
@pytest.mark.parametrize("name", ["t_poisson7_8", "t_elasticity_4", "t_filtered"])
def test_resumable_setup_matches_reference_setup(tmp_path, name):
    # tools/setup_resumable.py replays amgkit.setup's loop body level by level,
    # pickling each finished level; a run interrupted after level 1 and resumed
    # must give the reference's hierarchy bit for bit
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from setup_resumable import setup_resumable
    from amgkit import AmgConfig, SparseMatrix, setup

    if name == "t_poisson7_8":
        a0 = problems.poisson7(8, 8, 8)
        cfg = dict(smoother="fsai")
    elif name == "t_elasticity_4":
        a0, coords = problems.elasticity3d(4, 4, 4, sigma=1.0, nu=0.3, seed=1)
        cfg = dict(smoother="fsai", interp="bamg", testspace="rigid_body", n_test_vectors=6, coords=coords)
    else:  # operator filtering: nonsymmetric coarse levels, LU coarsest factor
        a0 = problems.poisson7(6, 6, 6)
        cfg = dict(smoother="jacobi", filter_target="operator", filter_rho=0.5, max_coarse=20)
    A = SparseMatrix(a0.nrows, a0.ncols, a0.row_offsets, a0.col_indices, a0.values, check=True)
    want = setup(A, AmgConfig(**cfg))
    st = str(tmp_path / "state")
    full = setup_resumable(A, AmgConfig(**cfg), st)
    # interrupted run: keep only the first finished level, resume
    st2 = str(tmp_path / "state2")
    os.makedirs(st2)
    import shutil

    shutil.copy(os.path.join(st, "level_0.pkl"), st2)
    resumed = setup_resumable(A, AmgConfig(**cfg), st2)
    for h in (full, resumed):
        assert h.n_levels == want.n_levels and h.factor_kind == want.factor_kind and h.symmetric == want.symmetric
        for l1, l2 in zip(h.levels, want.levels):
            assert hiercache.csr_digest(l1.a) == hiercache.csr_digest(l2.a)
            for f in ("p", "pt"):
                m1, m2 = getattr(l1, f), getattr(l2, f)
                assert (m1 is None) == (m2 is None)
                if m1 is not None:
                    assert hiercache.csr_digest(m1) == hiercache.csr_digest(m2)
            if l2.smoother is not None:
                assert l1.smoother.omega == l2.smoother.omega
                if l2.smoother.kind == "fsai":
                    assert hiercache.csr_digest(l1.smoother.gmat) == hiercache.csr_digest(l2.smoother.gmat)
        np.testing.assert_array_equal(np.asarray(h.factor[0]), np.asarray(want.factor[0]))
