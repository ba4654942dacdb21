"""Pin the CPU oracle against the reference's own outputs (golden vectors).

The oracle restates the reference with the same numpy / scipy calls, so on
the same numpy / scipy build it must reproduce every golden vector bit for
bit; the plain-C row-sum restatement must match np.add.reduceat bit for bit.
"""
import ctypes
import os

import numpy as np
import pytest

from golden_io import HIER_CASES, SPMV_CASES, cases_with, load_case, load_spmv_case, matrices_of
from oracle import solve as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", HIER_CASES)
def test_oracle_kernels_match_reference_bitwise(name):
    c = load_case(name)
    h, vec = c["h"], c["vec"]
    for k, slot, m in matrices_of(h):
        x = vec[f"spmv_L{k}_{slot}_x"]
        np.testing.assert_array_equal(O.spmv(m, x), vec[f"spmv_L{k}_{slot}_y"], err_msg=f"L{k}.{slot}")
    for k, lvl in enumerate(h.levels[:-1]):
        b, x0 = vec[f"smooth_L{k}_b"], vec[f"smooth_L{k}_x0"]
        for steps in (1, 2):
            np.testing.assert_array_equal(
                O.apply_smoother(lvl.smoother, lvl.a, b, np.zeros_like(b), steps), vec[f"smooth_L{k}_zero_{steps}"])
            np.testing.assert_array_equal(
                O.apply_smoother(lvl.smoother, lvl.a, b, x0, steps), vec[f"smooth_L{k}_x0_{steps}"])
    np.testing.assert_array_equal(O.coarse_solve(h, vec["coarse_y"]), vec["coarse_z"])
    np.testing.assert_array_equal(O.vcycle(h, vec["y"]), vec["vcycle_z"])


@pytest.mark.parametrize("name", cases_with("pcg"))
def test_oracle_pcg_matches_reference(name):
    c = load_case(name)
    h, vec, exp = c["h"], c["vec"], c["expect"]["pcg"]
    a0 = h.levels[0].a
    res = O.pcg(lambda v: O.spmv(a0, v), vec["b"], apply_m=lambda r: O.vcycle(h, r),
                config=O.KrylovConfig(rtol=exp["rtol"], max_iters=exp["max_iters"], record_history=True))
    assert res.n_iterations == exp["n_iterations"]
    assert res.converged == exp["converged"]
    np.testing.assert_allclose(res.x, vec["pcg_x"], rtol=0, atol=1e-13 * np.abs(vec["pcg_x"]).max())
    np.testing.assert_allclose([r for _, r in res.history], exp["history"], rtol=1e-12)


def _crowsum():
    lib = os.path.join(ROOT, "oracle", "build", "liboracle_rowsum.so")
    if not os.path.exists(lib):
        from paper_2102_07417_b200 import build

        build.build_oracle()
    return ctypes.CDLL(lib)


@pytest.mark.parametrize("name", SPMV_CASES)
def test_c_rowsum_restatement_is_bitwise_reference_order(name):
    m, x, y = load_spmv_case(name)
    L = _crowsum()
    out = np.empty(m.nrows)
    scratch = np.empty(max(1, int(np.diff(m.row_offsets).max(initial=1))))
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    L.oracle_csr_spmv(ctypes.c_int64(m.nrows), P(m.row_offsets), P(m.col_indices), P(m.values), P(x), P(out),
                      P(scratch))
    np.testing.assert_array_equal(out, y)
    np.testing.assert_array_equal(O.spmv(m, x), y)


def test_c_rowsum_random_lengths_match_reduceat():
    rng = np.random.default_rng(1)
    lens = np.concatenate([np.arange(0, 300), rng.integers(0, 2000, 100)])
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    data = rng.standard_normal(off[-1]) * 10.0 ** rng.integers(-8, 8, off[-1])
    out = np.empty(lens.size)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _crowsum().oracle_segment_sums(ctypes.c_int64(lens.size), P(off), P(data), P(out))
    np.testing.assert_array_equal(out, O.row_segment_sums(data, off))


def test_oracle_pcg_edge_cases():
    c = load_case("poisson7_12")
    h = c["h"]
    a0 = h.levels[0].a
    A = lambda v: O.spmv(a0, v)
    M = lambda r: O.vcycle(h, r)
    z = O.pcg(A, np.zeros(a0.nrows), apply_m=M)
    assert z.converged and z.n_iterations == 0 and z.relres == 0.0 and not z.x.any()
    xs = np.random.default_rng(3).standard_normal(a0.nrows)
    r = O.pcg(A, A(xs), apply_m=M, x0=xs)
    assert r.converged and r.n_iterations == 0
    with pytest.raises(O.NotSpdError, match="curvature"):
        O.pcg(lambda v: -A(v), c["b"], apply_m=M)
    r = O.pcg(A, c["b"], apply_m=M, config=O.KrylovConfig(rtol=1e-14, max_iters=3))
    assert not r.converged and r.n_iterations == 3


@pytest.mark.parametrize("name", ["poisson2d_12_lu", "poisson7_12_bicg"])
def test_oracle_bicgstab_matches_reference(name):
    c = load_case(name)
    h, vec, exp = c["h"], c["vec"], c["expect"]["bicgstab"]
    a0 = h.levels[0].a
    res = O.bicgstab(lambda v: O.spmv(a0, v), vec["b"], apply_m=lambda r: O.vcycle(h, r),
                     config=O.KrylovConfig(rtol=exp["rtol"], max_iters=exp["max_iters"], record_history=True))
    assert res.n_iterations == exp["n_iterations"] and res.converged == exp["converged"]
    assert res.restarts == exp["restarts"]
    np.testing.assert_allclose(res.x, vec["bicgstab_x"], rtol=0, atol=1e-13 * np.abs(vec["bicgstab_x"]).max())
