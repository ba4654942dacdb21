"""On-disk hierarchy cache: the setup output the solve path consumes.

Hierarchy setup (coarsening, interpolation, FSAI, Galerkin products) stays in
the reference's host Python (``amgkit/hierarchy.py:155-223``).  Setup is
expensive (minutes to hours for the BASELINE configs) and the
reference is not importable on the GPU box, so ``tools/export_hierarchy.py``
runs ``amgkit.setup`` once in the build container and freezes the result here.

The in-memory form is a duck-typed mirror of ``AmgHierarchy`` / ``Level`` /
``Smoother`` (``amgkit/hierarchy.py:95-152``, ``amgkit/smoothers.py:26-43``)
so that :meth:`DeviceHierarchy.from_reference` accepts either.

Three storage modes:

* ``full``: every level's A, P, Pt, G, Gt is stored.
* ``compact``: only what setup *chose* is stored -- G and P per level, the
  relaxation factors and the coarsest factor.  A_0 is rebuilt from the
  generator (``problems.py``), A_{k+1} by the Galerkin product, Pt and Gt by
  exact transposes, each restating the reference's own producer
  (``amgkit/sparse.py:220-224, 256-282``) with the same scipy calls, and then
  verified against SHA-256 digests of the reference's arrays recorded at
  export time.  Any mismatch raises: a hierarchy that differs from the
  reference's is never used silently.
* ``lean``: ``compact`` without the FSAI coefficients.  Only G's final
  sparsity pattern (and the rows that fell back to Jacobi) is stored; the
  coefficients are a pure function of (A_k, pattern) -- one dense Cholesky
  solve per row, ``amgkit/smoothers.py:80-96`` -- and are replayed with the
  same LAPACK routines scipy calls (``csrc/fsai_host.c``), then checked
  against the digest of the reference's G.  This is what makes the
  16.8 M-row config-4 hierarchy shippable (its level-1 G alone holds 33 M
  distinct fp64 coefficients).
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass, field

import numpy as np

from .problems import Csr, build_config

__all__ = [
    "HostSmoother",
    "HostLevel",
    "HostHierarchy",
    "save_hierarchy",
    "load_hierarchy",
    "csr_digest",
    "galerkin_product",
    "transpose",
    "galerkin_product_device",
    "transpose_device",
]

FORMAT = "amgb200-hier-v1"
MODES = ("full", "compact", "lean")


@dataclass
class HostSmoother:
    """Mirror of ``amgkit.smoothers.Smoother`` (fields the solve path reads)."""

    kind: str
    omega: float = 1.0
    gmat: Csr | None = None
    gmat_t: Csr | None = None
    inv_diag: np.ndarray | None = None


@dataclass
class HostLevel:
    """Mirror of ``amgkit.hierarchy.Level``."""

    a: Csr
    smoother: HostSmoother | None = None
    p: Csr | None = None
    pt: Csr | None = None


@dataclass
class _Cycle:
    nu1: int = 1
    nu2: int = 1


@dataclass
class HostHierarchy:
    """Mirror of ``amgkit.hierarchy.AmgHierarchy`` after setup."""

    levels: list
    config: _Cycle
    factor: tuple
    factor_kind: str
    symmetric: bool = True
    meta: dict = field(default_factory=dict)

    @property
    def n_levels(self):
        return len(self.levels)


def _as_csr(m):
    return Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def csr_digest(m):
    h = hashlib.sha256()
    h.update(np.asarray([m.nrows, m.ncols], dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(m.row_offsets, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(m.col_indices, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(m.values, dtype=np.float64).tobytes())
    return h.hexdigest()


def _from_scipy(m):
    # restates SparseMatrix.from_scipy (amgkit/sparse.py:134-140)
    m = m.tocsr()
    if not m.has_canonical_format:
        m.sum_duplicates()
    m.sort_indices()
    return Csr(m.shape[0], m.shape[1], m.indptr, m.indices, m.data)


def _to_scipy(a):
    import scipy.sparse as sp

    return sp.csr_matrix((a.values, a.col_indices, a.row_offsets), shape=(a.nrows, a.ncols))


def transpose(a):
    """Exact transpose; restates ``amgkit/sparse.py:220-224``."""
    t = _to_scipy(a).transpose().tocsr()
    t.sort_indices()
    return _from_scipy(t)


def galerkin_product(a, p, symmetrize):
    """P^T A P with optional (R + R^T)/2; restates ``amgkit/sparse.py:256-282``."""
    import scipy.sparse as sp

    ps = _to_scipy(p)
    r = ps.T @ (_to_scipy(a) @ ps)
    if symmetrize:
        r = (r + r.T) * 0.5
    r = sp.csr_matrix(r)
    r.sum_duplicates()
    r.sort_indices()
    r.eliminate_zeros()
    return _from_scipy(r)


def _device_result(handle):
    """Copy an ``amg_csr_result_t`` into a :class:`Csr` and free it."""
    import ctypes

    from . import _capi

    L = _capi.lib()
    try:
        nr, nc, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _capi.check(L.amg_csr_result_shape(handle, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nnz)))
        off = np.empty(nr.value + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int32)
        val = np.empty(nnz.value, dtype=np.float64)
        _capi.check(L.amg_csr_result_fetch(handle, _capi.ptr(off), _capi.ptr(col), _capi.ptr(val)))
    finally:
        L.amg_csr_result_free(handle)
    return Csr(nr.value, nc.value, off, col, val)


def transpose_device(a, device=0):
    """:func:`transpose` on the GPU (``amg_device_transpose``), bit-identical."""
    import ctypes

    from . import _capi

    out = ctypes.c_void_p()
    _capi.check(_capi.lib().amg_device_transpose(
        int(device), a.nrows, a.ncols, _capi.ptr(a.row_offsets), _capi.ptr(a.col_indices), _capi.ptr(a.values),
        ctypes.byref(out)), "amg_device_transpose")
    return _device_result(out)


def galerkin_product_device(a, p, symmetrize, device=0):
    """:func:`galerkin_product` on the GPU (``amg_device_galerkin``): the same terms added in
    the same order as scipy's row-by-row SpGEMM, so the result is bit-identical."""
    import ctypes

    from . import _capi

    if a.nrows != a.ncols or a.ncols != p.nrows:
        raise ValueError("galerkin_product_device: shapes do not chain")
    out = ctypes.c_void_p()
    _capi.check(_capi.lib().amg_device_galerkin(
        int(device), a.nrows, p.ncols, _capi.ptr(a.row_offsets), _capi.ptr(a.col_indices), _capi.ptr(a.values),
        _capi.ptr(p.row_offsets), _capi.ptr(p.col_indices), _capi.ptr(p.values), 1 if symmetrize else 0,
        ctypes.byref(out)), "amg_device_galerkin")
    return _device_result(out)


def _save_csr(path, m):
    np.savez_compressed(path, shape=np.asarray([m.nrows, m.ncols], dtype=np.int64),
             row_offsets=np.asarray(m.row_offsets, dtype=np.int64),
             col_indices=np.asarray(m.col_indices, dtype=np.int32),
             values=np.asarray(m.values, dtype=np.float64))


def _load_csr(path):
    with np.load(path) as z:
        nr, nc = (int(v) for v in z["shape"])
        return Csr(nr, nc, z["row_offsets"], z["col_indices"], z["values"])


def _save_csr_packed(path, m):
    """CSR with row lengths and delta-coded columns (lean mode; deflates ~2x better)."""
    lens = np.diff(np.asarray(m.row_offsets, dtype=np.int64))
    d = np.diff(np.asarray(m.col_indices, dtype=np.int64), prepend=0).astype(np.int32)
    lt = np.uint8 if lens.size == 0 or lens.max() < 256 else np.int32
    np.savez_compressed(path, shape=np.asarray([m.nrows, m.ncols], dtype=np.int64), lens=lens.astype(lt),
                        dcols=d, values=np.asarray(m.values, dtype=np.float64))


def _load_csr_any(path):
    with np.load(path) as z:
        if "dcols" not in z.files:
            nr, nc = (int(v) for v in z["shape"])
            return Csr(nr, nc, z["row_offsets"], z["col_indices"], z["values"])
        nr, nc = (int(v) for v in z["shape"])
        offs = np.zeros(nr + 1, dtype=np.int64)
        np.cumsum(z["lens"].astype(np.int64), out=offs[1:])
        cols = np.cumsum(z["dcols"].astype(np.int64)).astype(np.int32)
        return Csr(nr, nc, offs, cols, z["values"])


def _save_pattern(path, g, fallback_mask=None):
    """G's sparsity only: row lengths and i - col per entry (small integers; deflates well)."""
    offs = np.asarray(g.row_offsets, dtype=np.int64)
    lens = np.diff(offs)
    rows = np.repeat(np.arange(g.nrows, dtype=np.int64), lens)
    rel = (rows - np.asarray(g.col_indices, dtype=np.int64)).astype(np.int32)
    if fallback_mask is None:
        fb = np.zeros(0, dtype=np.int64)
    else:
        fb = np.flatnonzero(np.asarray(fallback_mask, dtype=bool)).astype(np.int64)
    lt = np.uint8 if lens.size == 0 or lens.max() < 256 else np.int32
    np.savez_compressed(path, shape=np.asarray([g.nrows, g.ncols], dtype=np.int64), lens=lens.astype(lt),
                        rel=rel, fallback=fb)


def _fallback_mask(a, g):
    """Rows of G the reference reset to the Jacobi row (smoothers.py:94-97).

    The reference keeps only their count; they are identified by replaying
    every row and checking where the stored value is 1/sqrt(a_ii) instead of
    the Cholesky result.  Raises unless the replay then reproduces G exactly
    (a lean cache must rebuild the reference's G bit for bit).
    """
    from . import fsai_host

    ref = np.asarray(g.values, dtype=np.float64)
    vals = fsai_host.fsai_values(a, g.row_offsets, g.col_indices, None, allow_failed=True)
    same = vals == ref
    if same.all():
        return None
    lens = np.diff(np.asarray(g.row_offsets, dtype=np.int64))
    rows = np.unique(np.repeat(np.arange(g.nrows), lens)[~same])
    diag = _to_scipy(a).diagonal()
    mask = np.zeros(g.nrows, dtype=np.uint8)
    ok = (lens[rows] == 1) & (ref[g.row_offsets[rows]] == 1.0 / np.sqrt(diag[rows]))
    if not ok.all():
        raise ValueError(f"FSAI replay differs from the reference on row {int(rows[~ok][0])}: lean mode unusable")
    mask[rows] = 1
    vals = fsai_host.fsai_values(a, g.row_offsets, g.col_indices, mask)
    if not np.array_equal(vals, ref):
        raise ValueError("FSAI replay with the fallback rows does not reproduce the reference's G")
    return mask


def _load_pattern(path, a, threads=None):
    from . import fsai_host

    with np.load(path) as z:
        nr, nc = (int(v) for v in z["shape"])
        lens = z["lens"].astype(np.int64)
        rel = z["rel"].astype(np.int64)
        fb = z["fallback"]
    offs = np.zeros(nr + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    cols = (np.repeat(np.arange(nr, dtype=np.int64), lens) - rel).astype(np.int32)
    mask = None
    if fb.size:
        mask = np.zeros(nr, dtype=np.uint8)
        mask[fb] = 1
    vals = fsai_host.fsai_values(a, offs, cols, mask, threads=threads)
    return Csr(nr, nc, offs, cols, vals)


def save_hierarchy(h, directory, mode="full", generator=None, symmetrize_flags=None, extra=None):
    """Freeze a setup result (``amgkit.AmgHierarchy`` or :class:`HostHierarchy`).

    ``compact`` needs ``generator`` (a ``problems.CONFIGS`` name rebuilding
    A_0) and ``symmetrize_flags[k]`` -- the ``symmetrize`` argument setup
    passed to the Galerkin product of level k (``hierarchy.py:210``).
    """
    os.makedirs(directory, exist_ok=True)
    levels = h.levels
    man = {
        "format": FORMAT,
        "mode": mode,
        "generator": generator,
        "n_levels": len(levels),
        "nu1": int(h.config.nu1),
        "nu2": int(h.config.nu2),
        "symmetric": bool(h.symmetric),
        "factor_kind": h.factor_kind,
        "levels": [],
        "extra": extra or {},
    }
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    for k, lvl in enumerate(levels):
        ent = {"n": int(lvl.a.nrows), "nnz_a": int(lvl.a.nnz), "digest": {"a": csr_digest(lvl.a)}}
        if mode == "full" or (k == 0 and generator is None):
            # compact / lean rebuild A_0 from the named generator when there is one
            _save_csr(os.path.join(directory, f"L{k}_a.npz"), lvl.a)
        sm = lvl.smoother
        if sm is not None:
            ent["smoother"] = {"kind": sm.kind, "omega": float(sm.omega)}
            if sm.kind == "jacobi":
                np.save(os.path.join(directory, f"L{k}_invdiag.npy"), np.asarray(sm.inv_diag, dtype=np.float64))
            else:
                if mode == "lean":
                    _save_pattern(os.path.join(directory, f"L{k}_gpat.npz"), sm.gmat,
                                  _fallback_mask(lvl.a, sm.gmat))
                    ent["g_store"] = "pattern"
                else:
                    _save_csr(os.path.join(directory, f"L{k}_g.npz"), sm.gmat)
                ent["digest"]["g"] = csr_digest(sm.gmat)
                ent["digest"]["gt"] = csr_digest(sm.gmat_t)
                if mode == "full":
                    _save_csr(os.path.join(directory, f"L{k}_gt.npz"), sm.gmat_t)
        if lvl.p is not None:
            (_save_csr_packed if mode == "lean" else _save_csr)(os.path.join(directory, f"L{k}_p.npz"), lvl.p)
            ent["digest"]["p"] = csr_digest(lvl.p)
            ent["digest"]["pt"] = csr_digest(lvl.pt)
            if mode == "full":
                _save_csr(os.path.join(directory, f"L{k}_pt.npz"), lvl.pt)
            if symmetrize_flags is not None:
                ent["symmetrize_next"] = bool(symmetrize_flags[k])
        man["levels"].append(ent)
    fac = h.factor
    if h.factor_kind in ("cholesky", "cholesky+shift"):
        c, lower = fac
        if not lower:
            raise ValueError("expected a lower Cholesky factor (hierarchy.py:127)")
        np.save(os.path.join(directory, "coarse_c.npy"), np.tril(np.asarray(c, dtype=np.float64)))
    else:
        lu, piv = fac
        np.save(os.path.join(directory, "coarse_c.npy"), np.asarray(lu, dtype=np.float64))
        np.save(os.path.join(directory, "coarse_piv.npy"), np.asarray(piv, dtype=np.int32))
    with open(os.path.join(directory, "manifest.json"), "w") as f:
        json.dump(man, f, indent=1)
    return man


def load_hierarchy(directory, verify=True, threads=None, device=None):
    """Load a frozen hierarchy as a :class:`HostHierarchy`.

    ``device`` (a CUDA device index): rebuild the Galerkin products and the
    transposes with the library's device operators instead of scipy -- the
    same arrays bit for bit (digest-checked like the host path), several
    times faster on the multi-million-row configs.

    ``lean`` caches replay the FSAI coefficients on ``threads`` host threads
    (default: all available) and always verify them against the recorded
    digest of the reference's G (the replay is the one step whose result
    could depend on the host's LAPACK build).
    """
    with open(os.path.join(directory, "manifest.json")) as f:
        man = json.load(f)
    if man.get("format") != FORMAT:
        raise ValueError(f"{directory}: not an {FORMAT} hierarchy")
    mode = man["mode"]
    levels = []
    a = None
    for k, ent in enumerate(man["levels"]):
        if mode == "full" or (k == 0 and man.get("generator") is None):
            a = _load_csr(os.path.join(directory, f"L{k}_a.npz"))
        elif k == 0:
            a = build_config(man["generator"])
        else:
            prev = levels[k - 1]
            sym_next = man["levels"][k - 1].get("symmetrize_next", True)
            a = (galerkin_product_device(prev.a, prev.p, sym_next, device) if device is not None
                 else galerkin_product(prev.a, prev.p, sym_next))
        if verify and csr_digest(a) != ent["digest"]["a"]:
            raise ValueError(f"{directory}: level {k} operator does not match the reference digest")
        lvl = HostLevel(a=a)
        sm = ent.get("smoother")
        if sm is not None:
            if sm["kind"] == "jacobi":
                inv = np.load(os.path.join(directory, f"L{k}_invdiag.npy"))
                lvl.smoother = HostSmoother("jacobi", sm["omega"], inv_diag=inv)
            else:
                if ent.get("g_store") == "pattern":
                    g = _load_pattern(os.path.join(directory, f"L{k}_gpat.npz"), a, threads)
                    if csr_digest(g) != ent["digest"]["g"]:
                        raise ValueError(f"{directory}: level {k} replayed FSAI factor does not match the "
                                         "reference digest (host LAPACK differs from the export host's?)")
                else:
                    g = _load_csr(os.path.join(directory, f"L{k}_g.npz"))
                    if verify and "g" in ent["digest"] and csr_digest(g) != ent["digest"]["g"]:
                        raise ValueError(f"{directory}: level {k} G does not match the reference digest")
                gt_path = os.path.join(directory, f"L{k}_gt.npz")
                gt = (_load_csr(gt_path) if os.path.exists(gt_path)
                      else transpose_device(g, device) if device is not None else transpose(g))
                if verify and csr_digest(gt) != ent["digest"]["gt"]:
                    raise ValueError(f"{directory}: level {k} G^T does not match the reference digest")
                lvl.smoother = HostSmoother("fsai", sm["omega"], gmat=g, gmat_t=gt)
        p_path = os.path.join(directory, f"L{k}_p.npz")
        if os.path.exists(p_path):
            lvl.p = _load_csr_any(p_path)
            if verify and "p" in ent["digest"] and csr_digest(lvl.p) != ent["digest"]["p"]:
                raise ValueError(f"{directory}: level {k} P does not match the reference digest")
            pt_path = os.path.join(directory, f"L{k}_pt.npz")
            lvl.pt = (_load_csr(pt_path) if os.path.exists(pt_path)
                      else transpose_device(lvl.p, device) if device is not None else transpose(lvl.p))
            if verify and csr_digest(lvl.pt) != ent["digest"]["pt"]:
                raise ValueError(f"{directory}: level {k} P^T does not match the reference digest")
        levels.append(lvl)
    c = np.load(os.path.join(directory, "coarse_c.npy"))
    if man["factor_kind"] in ("cholesky", "cholesky+shift"):
        factor = (c, True)
    else:
        factor = (c, np.load(os.path.join(directory, "coarse_piv.npy")))
    return HostHierarchy(
        levels=levels,
        config=_Cycle(man["nu1"], man["nu2"]),
        factor=factor,
        factor_kind=man["factor_kind"],
        symmetric=man["symmetric"],
        meta=man,
    )
