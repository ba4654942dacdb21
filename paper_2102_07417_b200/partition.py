"""Row-block partition of every level across GPUs (one process per GPU).

The reference's only distribution model is DSMat-style row stripes
(``amgkit/striped.py:28-186``, ``PAPER.md:824-847``): contiguous balanced row
ranges (``partition_rows``, ``striped.py:28-41``) with per-neighbour column
blocks.  Here every level of the hierarchy is partitioned:

* level 0: ``partition_rows(n0, nranks)`` (for the structured configs the
  node order is x fastest, z slowest, so these are z-slabs);
* level k+1 inherits ownership from level k: coarse point c belongs to the
  rank owning its C-point (the fine row injecting into c -- coarse numbers
  follow ascending fine order, ``amgkit/sparse.py:185-189``), which keeps the
  ranges contiguous;
* from the agglomeration level k_a down the levels are REPLICATED: the
  restricted vector is all-gathered and every rank runs the rest of the
  V-cycle on the full (small) level, as Chronos does for its coarsest level
  (``PAPER.md:1308-1312``).

Each rank's local matrix keeps its rows and the *stored order of entries
within a row*; columns are renumbered to ``[0, n_own)`` for owned columns and
``n_own + i`` for the i-th halo column (sorted global id), so a local SpMV
sums every row in exactly the reference order -- distributed SpMV results are
bit-identical to the single-GPU ones.  Halo plans list, per peer, the owned
entries to send and the halo segment to receive.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .problems import Csr

__all__ = ["partition_rows", "HaloPlan", "LocalMatrix", "RankPlan", "plan_hierarchy"]


def partition_rows(n, nranks):
    """Balanced contiguous ranges; restates ``amgkit/striped.py:28-41``."""
    if nranks < 1:
        raise ValueError(f"need at least one stripe, got {nranks}")
    base, extra = divmod(int(n), nranks)
    sizes = np.full(nranks, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


@dataclass
class HaloPlan:
    """Exchange that fills ``x[n_own:n_own + n_halo]`` before a local SpMV."""

    n_own: int
    halo_cols: np.ndarray                   # sorted global ids (local index n_own + i)
    recv_peers: list = field(default_factory=list)
    recv_counts: list = field(default_factory=list)   # contiguous segments of halo_cols, by peer rank
    send_peers: list = field(default_factory=list)
    send_idx: list = field(default_factory=list)      # local owned indices sent to each peer

    @property
    def n_halo(self):
        return int(self.halo_cols.size)


@dataclass
class LocalMatrix:
    csr: Csr                 # local rows, local column ids
    halo: HaloPlan | None    # None: all columns local (replicated column space)
    row0: int                # global id of the first local row
    global_shape: tuple


@dataclass
class RankPlan:
    rank: int
    nranks: int
    starts: list             # per level: int64[nranks + 1] row ranges
    agglom_level: int        # first replicated level (n_levels - 1 at most)
    mats: dict               # (level, slot) -> LocalMatrix
    smoothers: dict          # level -> (kind, omega, local inv_diag or None)
    factor: tuple
    factor_kind: str
    nu1: int
    nu2: int

    def n_local(self, level):
        if level >= self.agglom_level:
            return int(self.starts[level][-1])
        s = self.starts[level]
        return int(s[self.rank + 1] - s[self.rank])


def _coarse_starts(p, fine_starts):
    """Inherit ownership of the coarse points of P from the fine partition."""
    n, nc = p.nrows, p.ncols
    off = p.row_offsets
    lens = np.diff(off)
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    # home fine row of each coarse column: its injection row (single entry 1.0),
    # else the row holding the largest |P| entry of the column
    home = np.full(nc, -1, dtype=np.int64)
    inj = (lens[rows] == 1) & (p.values == 1.0)
    ci = p.col_indices[inj].astype(np.int64)
    ri = rows[inj]
    first = np.full(nc, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(first, ci, ri)
    has = first != np.iinfo(np.int64).max
    home[has] = first[has]
    if not has.all():
        order = np.lexsort((-np.abs(p.values), p.col_indices))
        cols_sorted = p.col_indices[order]
        firsts = np.concatenate([[True], cols_sorted[1:] != cols_sorted[:-1]])
        best_rows = rows[order][firsts]
        best_cols = cols_sorted[firsts].astype(np.int64)
        miss = ~has[best_cols]
        home[best_cols[miss]] = best_rows[miss]
    owner = np.searchsorted(fine_starts, home, side="right") - 1
    if np.all(np.diff(owner) >= 0):
        counts = np.bincount(owner, minlength=len(fine_starts) - 1)
        return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return partition_rows(nc, len(fine_starts) - 1)  # not monotone: balanced ranges


def _localize(m, row_starts, col_starts, rank, replicated_cols):
    """Local rows of ``m`` with renumbered columns + the halo plan of ``rank``."""
    nr = len(row_starts) - 1
    r0, r1 = int(row_starts[rank]), int(row_starts[rank + 1])
    off = m.row_offsets
    k0, k1 = int(off[r0]), int(off[r1])
    cols = m.col_indices[k0:k1].astype(np.int64)
    loff = (off[r0:r1 + 1] - k0).astype(np.int64)
    vals = m.values[k0:k1]
    if replicated_cols:
        return LocalMatrix(Csr(r1 - r0, m.ncols, loff, cols.astype(np.int32), vals), None, r0, m.shape)
    c0, c1 = int(col_starts[rank]), int(col_starts[rank + 1])
    own = (cols >= c0) & (cols < c1)
    halo = np.unique(cols[~own])
    local = np.empty_like(cols)
    local[own] = cols[own] - c0
    local[~own] = (c1 - c0) + np.searchsorted(halo, cols[~own])
    plan = HaloPlan(n_own=c1 - c0, halo_cols=halo)
    owner = np.searchsorted(col_starts, halo, side="right") - 1
    for q in range(nr):
        cnt = int(np.sum(owner == q))
        if cnt:
            plan.recv_peers.append(q)
            plan.recv_counts.append(cnt)
    # what every other rank needs from me (each rank sees the global matrix)
    for q in range(nr):
        if q == rank:
            continue
        qr0, qr1 = int(row_starts[q]), int(row_starts[q + 1])
        qc = m.col_indices[int(off[qr0]):int(off[qr1])].astype(np.int64)
        need = np.unique(qc[(qc >= c0) & (qc < c1)])
        qc0, qc1 = int(col_starts[q]), int(col_starts[q + 1])
        need = need[(need < qc0) | (need >= qc1)]
        if need.size:
            plan.send_peers.append(q)
            plan.send_idx.append((need - c0).astype(np.int32))
    return LocalMatrix(Csr(r1 - r0, (c1 - c0) + halo.size, loff, local.astype(np.int32), vals), plan, r0, m.shape)


def interior_range(csr, n_own, align=128):
    """Rows [lo, hi) of a local matrix that touch no halo column (column >= n_own).

    Mirrors ``interior_range`` in csrc/capi.cu: lo = 1 + the last halo-touching
    row in the first half, hi = the first halo-touching row in the second half,
    aligned inwards to ``align`` rows; (0, 0) when that leaves fewer than
    max(align, n / 8) rows.  The device runs the interior rows while the halo
    is in flight, the boundary rows [0, lo) + [hi, n) after it arrived.
    """
    n = csr.nrows
    offs = np.asarray(csr.row_offsets, dtype=np.int64)
    rows = np.repeat(np.arange(n), np.diff(offs))
    touch = np.zeros(n, dtype=bool)
    touch[rows[np.asarray(csr.col_indices) >= n_own]] = True
    lo_rows = np.flatnonzero(touch[: n // 2])
    hi_rows = np.flatnonzero(touch[n // 2:])
    lo_end = int(lo_rows[-1]) + 1 if lo_rows.size else 0
    hi_start = int(hi_rows[0]) + n // 2 if hi_rows.size else n
    a = (lo_end + align - 1) // align * align
    b = hi_start // align * align
    if b - a >= align and b - a >= n // 8:
        return a, b
    return 0, 0


def plan_hierarchy(h, nranks, rank, agglom_rows=4096):
    """Partition plan of ``rank`` for hierarchy ``h`` (identical inputs on every rank).

    ``agglom_rows``: levels with at most this many global rows (and all
    coarser ones) are replicated.  The coarsest level is always replicated.
    """
    levels = h.levels
    nl = len(levels)
    starts = [partition_rows(levels[0].a.nrows, nranks)]
    for k in range(nl - 1):
        starts.append(_coarse_starts(levels[k].p, starts[k]))
    ka = nl - 1
    for k in range(1, nl):
        if levels[k].a.nrows <= agglom_rows:
            ka = k
            break
    if nranks == 1:
        ka = nl  # nothing replicated beyond the usual coarse solve
    mats, smoothers = {}, {}
    full = lambda n: np.array([0] + [n] * nranks, dtype=np.int64)
    for k, lv in enumerate(levels):
        rep = k >= ka
        rs = full(lv.a.nrows) if rep else starts[k]
        # replicated: every rank owns all rows -> localize as rank 0 of a 1-rank split
        if rep:
            mats[(k, "a")] = _localize(lv.a, np.array([0, lv.a.nrows]), None, 0, True)
        else:
            mats[(k, "a")] = _localize(lv.a, rs, starts[k], rank, False)
        if lv.p is None:
            continue
        crep = (k + 1) >= ka
        if rep:
            mats[(k, "p")] = _localize(lv.p, np.array([0, lv.p.nrows]), None, 0, True)
            mats[(k, "pt")] = _localize(lv.pt, np.array([0, lv.pt.nrows]), None, 0, True)
        else:
            mats[(k, "p")] = _localize(lv.p, starts[k], starts[k + 1], rank, crep)
            mats[(k, "pt")] = _localize(lv.pt, starts[k + 1], starts[k], rank, False)
        sm = lv.smoother
        if sm.kind == "fsai":
            for slot, m in (("g", sm.gmat), ("gt", sm.gmat_t)):
                if rep:
                    mats[(k, slot)] = _localize(m, np.array([0, m.nrows]), None, 0, True)
                else:
                    mats[(k, slot)] = _localize(m, starts[k], starts[k], rank, False)
            smoothers[k] = ("fsai", float(sm.omega), None)
        else:
            inv = np.asarray(sm.inv_diag) if rep else np.asarray(sm.inv_diag)[starts[k][rank]:starts[k][rank + 1]]
            smoothers[k] = ("jacobi", float(sm.omega), inv)
    return RankPlan(rank=rank, nranks=nranks, starts=starts, agglom_level=min(ka, nl),
                    mats=mats, smoothers=smoothers, factor=h.factor, factor_kind=h.factor_kind,
                    nu1=int(h.config.nu1), nu2=int(h.config.nu2))
