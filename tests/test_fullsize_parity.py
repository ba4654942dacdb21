"""Parity at the BASELINE sizes (configs 1-4) on the frozen reference
hierarchies tracked in hier_cache/ (a missing cache FAILS: it ships with the
repository, lean mode, see hiercache.py).

* every matrix of the first levels: device SpMV bit-identical to the oracle;
* one V-cycle within 1e-12 of the oracle (test_acceptance.py:53-57 metric);
* PCG: iteration count within +-1 of the REFERENCE's own solve recorded at
  export (amgkit pcg on the same hierarchy and RHS), device-reported relres
  equal to the true residual of the returned x, and <= rtol;
* size-independent properties: V-cycle linearity and symmetry.
"""
import os

import numpy as np
import pytest

from conftest import _relerr

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CACHE = os.path.join(ROOT, "hier_cache")
CONFIGS = ["c1_poisson7_64", "c2_hetero27_128", "c3_elasticity_64", "c4_rtanis7_256"]
# caches that may legitimately be absent from a snapshot (everything else must ship)
OPTIONAL = {}
# the opt-in tail variants re-upload the hierarchy: skipped above this many rows (config 4: 16.8 M)
VARIANT_MAX_ROWS = 4_000_000


def _load(name):
    d = os.path.join(CACHE, name)
    if not os.path.exists(os.path.join(d, "manifest.json")):
        if name in OPTIONAL:
            pytest.skip(f"{name}: hierarchy cache not in this snapshot ({OPTIONAL[name]})")
        pytest.fail(f"{name}: hierarchy cache {d} missing (it is tracked in git; run tools/export_hierarchy.py)")
    from paper_2102_07417_b200 import hiercache

    return hiercache.load_hierarchy(d, verify=True)


@pytest.fixture(scope="module", params=CONFIGS)
def full(request):
    import paper_2102_07417_b200 as amg

    h = _load(request.param)
    dh = amg.DeviceHierarchy.from_reference(h)
    yield request.param, h, dh
    dh.close()


def test_fullsize_spmv_bit_identical(full):
    from oracle import solve as O

    name, h, dh = full
    rng = np.random.default_rng(17)
    for k, lv in enumerate(h.levels[:2]):
        mats = {"a": lv.a}
        if lv.p is not None:
            mats.update(p=lv.p, pt=lv.pt, g=lv.smoother.gmat, gt=lv.smoother.gmat_t)
        for slot, m in mats.items():
            x = rng.uniform(-1, 1, m.ncols)
            np.testing.assert_array_equal(dh.matrix(k, slot)(x), O.spmv(m, x), err_msg=f"{name} L{k}.{slot}")


def test_fullsize_vcycle_and_properties(full):
    from oracle import solve as O

    name, h, dh = full
    n = h.levels[0].a.nrows
    rng = np.random.default_rng(5)
    y1, y2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    z1 = dh.vcycle(y1)
    assert _relerr(z1, O.vcycle(h, y1)) <= 1e-12
    z2 = dh.vcycle(y2)
    lin = dh.vcycle(2.0 * y1 - 3.0 * y2)
    assert _relerr(lin, 2.0 * z1 - 3.0 * z2) <= 1e-11
    assert abs(z1 @ y2 - y1 @ z2) <= 1e-10 * np.linalg.norm(z1) * np.linalg.norm(y2)


def test_fullsize_pcg_matches_reference_solve(full):
    import paper_2102_07417_b200 as amg
    from oracle import solve as O
    from paper_2102_07417_b200 import problems

    name, h, dh = full
    ref = h.meta.get("extra", {}).get("reference_solve")
    b = problems.build_rhs(name, h.levels[0].a.nrows)
    res = amg.pcg(dh.A0, b, apply_m=dh.vcycle, config=amg.KrylovConfig(rtol=1e-8, record_history=True))
    assert res.converged and res.relres <= 1e-8
    true = np.linalg.norm(b - O.spmv(h.levels[0].a, res.x)) / np.linalg.norm(b)
    assert res.relres == pytest.approx(true, rel=1e-6)
    if ref is not None:
        assert abs(res.n_iterations - ref["n_iterations"]) <= 1
        m = min(len(ref["history"]), len(res.history))
        np.testing.assert_allclose([r for _, r in res.history[:m]], ref["history"][:m], rtol=1e-6, atol=1e-12)
    # run-to-run bitwise determinism at full size
    res2 = amg.pcg(dh.A0, b, apply_m=dh.vcycle, config=amg.KrylovConfig(rtol=1e-8, record_history=True))
    np.testing.assert_array_equal(res.x, res2.x)


def test_fullsize_tail_dsm_bit_identical(full):
    # the cluster tail with its level vectors in distributed shared memory
    import paper_2102_07417_b200 as amg

    name, h, dh = full
    if h.levels[0].a.nrows > VARIANT_MAX_ROWS:
        pytest.skip("opt-in variant: checked on configs 1-3")
    dh2 = amg.DeviceHierarchy.from_reference(h, options={"tail_dsm": 1})
    y = np.random.default_rng(31).uniform(-1, 1, h.levels[0].a.nrows)
    np.testing.assert_array_equal(dh2.vcycle(y), dh.vcycle(y))
    dh2.close()


def test_fullsize_wider_tail_bit_identical(full):
    # a cluster tail that starts one level higher, its SpMV blocks run in product chunks
    import paper_2102_07417_b200 as amg

    name, h, dh = full
    if h.levels[0].a.nrows > VARIANT_MAX_ROWS:
        pytest.skip("opt-in variant: checked on configs 1-3")
    dh2 = amg.DeviceHierarchy.from_reference(h, options={"tail_nnz": 2_000_000, "tail_pcap": 4096})
    y = np.random.default_rng(37).uniform(-1, 1, h.levels[0].a.nrows)
    np.testing.assert_array_equal(dh2.vcycle(y), dh.vcycle(y))
    dh2.close()
