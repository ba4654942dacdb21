"""Device Galerkin product / transpose against the reference's scipy path.

``hiercache.galerkin_product`` / ``transpose`` restate ``amgkit/sparse.py:256-282, 220-224``
with the reference's own scipy calls (pinned bitwise against amgkit by test_hiercache.py);
the device operators must reproduce them bit for bit: same terms, same order, exact zeros
dropped, canonical CSR out.
"""
import os

import numpy as np
import pytest

from golden_io import HIER_CASES, load_case
from paper_2102_07417_b200 import hiercache
from paper_2102_07417_b200.problems import Csr

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _same(x, y):
    assert (x.nrows, x.ncols) == (y.nrows, y.ncols)
    np.testing.assert_array_equal(x.row_offsets, y.row_offsets)
    np.testing.assert_array_equal(x.col_indices, y.col_indices)
    assert x.values.tobytes() == y.values.tobytes()  # bit for bit, signed zeros included


@pytest.mark.parametrize("name", HIER_CASES)
def test_device_galerkin_and_transpose_match_scipy_on_golden_hierarchies(name):
    h = load_case(name)["h"]
    for lv in h.levels:
        if lv.p is None:
            continue
        for sym in (True, False):
            _same(hiercache.galerkin_product_device(lv.a, lv.p, sym), hiercache.galerkin_product(lv.a, lv.p, sym))
        _same(hiercache.transpose_device(lv.p), hiercache.transpose(lv.p))
        if lv.smoother is not None and lv.smoother.gmat is not None:
            _same(hiercache.transpose_device(lv.smoother.gmat), hiercache.transpose(lv.smoother.gmat))
        _same(hiercache.transpose_device(lv.a), hiercache.transpose(lv.a))


def _random_csr(rng, nrows, ncols, density, integer):
    import scipy.sparse as sp

    m = sp.random(nrows, ncols, density=density, format="csr", random_state=rng,
                  data_rvs=(lambda k: rng.integers(-2, 3, k).astype(float)) if integer else None)
    m.sort_indices()
    return Csr(nrows, ncols, m.indptr, m.indices, m.data)


@pytest.mark.parametrize("integer", [False, True])
def test_device_galerkin_random_with_cancellation_and_empty_rows(integer):
    # integer values: sums cancel to exact zeros (dropped, like scipy), explicit zeros in the
    # inputs; sparse P: coarse columns nobody interpolates to, fine rows without entries
    rng = np.random.default_rng(5)
    for n, m, da, dp in [(400, 90, 0.03, 0.02), (257, 33, 0.05, 0.01), (64, 64, 0.2, 0.1), (50, 1, 0.1, 0.5)]:
        a = _random_csr(rng, n, n, da, integer)
        p = _random_csr(rng, n, m, dp, integer)
        for sym in (True, False):
            _same(hiercache.galerkin_product_device(a, p, sym), hiercache.galerkin_product(a, p, sym))
        _same(hiercache.transpose_device(p), hiercache.transpose(p))


def test_device_setup_empty_matrix():
    z = Csr(5, 5, np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    p = Csr(5, 2, np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    _same(hiercache.galerkin_product_device(z, p, True), hiercache.galerkin_product(z, p, True))
    _same(hiercache.transpose_device(p), hiercache.transpose(p))


@pytest.mark.parametrize("name", ["c1_poisson7_64", "c2_hetero27_128"])
def test_lean_cache_loads_through_the_device_operators(name):
    # every Galerkin product and transpose of the frozen hierarchy rebuilt on the GPU and checked
    # against the SHA-256 digests of the reference's own arrays (load_hierarchy raises on a mismatch)
    d = os.path.join(ROOT, "hier_cache", name)
    if not os.path.exists(os.path.join(d, "manifest.json")):
        pytest.fail(f"{name}: hierarchy cache missing (tracked in git)")
    h = hiercache.load_hierarchy(d, verify=True, device=0)
    assert h.n_levels == len(h.meta["levels"])
