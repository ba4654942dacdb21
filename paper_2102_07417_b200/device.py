"""Device-resident hierarchy: the upload side of the drop-in boundary.

``DeviceHierarchy.from_reference(h)`` takes the reference's setup output --
an ``amgkit.AmgHierarchy`` (``amgkit/hierarchy.py:108-152``) or the
duck-typed :class:`~paper_2102_07417_b200.hiercache.HostHierarchy` loaded from
a frozen cache -- and uploads, once, every level's A, P, P^T, FSAI G / G^T
(or Jacobi inverse diagonal), the relaxation factors omega_k, the cycle
counts nu1 / nu2 and the coarsest factor (``np.tril(c)`` of the lower
Cholesky factor, or LU + pivots) through the C ABI.

Its members are the device operators the shim's ``pcg`` / ``vcycle`` /
``spmv`` accept in place of the reference's callables:

* ``dh.A0``      -- level-0 operator, ``dh.A0(x)`` = ``amgkit.spmv(A0, x)``
* ``dh.vcycle``  -- preconditioner, ``dh.vcycle(r)`` = ``amgkit.vcycle(h, r)``
* ``dh.matrix(level, "a"|"p"|"pt"|"g"|"gt")`` -- any uploaded matrix
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _capi as C
from .errors import AmgError, DimensionMismatchError

__all__ = ["DeviceHierarchy", "DeviceMatrix", "DeviceVcycle", "model_bytes_flops", "layout_bytes_per_iter",
           "nccl_unique_id"]


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0 makes it, every rank passes it to from_plan)."""
    buf = ctypes.create_string_buffer(128)
    C.check(C.lib().amg_nccl_unique_id(buf), "amg_nccl_unique_id")
    return buf.raw


def _host_f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _is_cuda_tensor(x):
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


class DeviceSmoother:
    """Level smoother handle: what ``Level.smoother`` is to the reference's ``apply_smoother``."""

    def __init__(self, dh, level):
        self.dh = dh
        self.level = level


class DeviceMatrix:
    """A matrix slot of the device hierarchy; calling it is ``spmv``."""

    def __init__(self, dh, level, slot, nrows, ncols, nnz):
        self.dh = dh
        self.level = level
        self.slot = slot
        self.nrows = nrows
        self.ncols = ncols
        self.nnz = nnz

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def __call__(self, x):
        return self.dh.spmv(self.level, self.slot, x)

    def __repr__(self):
        return f"DeviceMatrix(level={self.level}, slot={self.slot!r}, {self.nrows}x{self.ncols}, nnz={self.nnz})"


class DeviceVcycle:
    """``vcycle(h, .)`` on the device; calling it applies one V-cycle."""

    def __init__(self, dh):
        self.dh = dh

    def __call__(self, y):
        return self.dh.apply_vcycle(y)


class DeviceHierarchy:
    """Uploaded hierarchy bound to one GPU (one rank)."""

    def __init__(self, device=0, rank=0, nranks=1, nccl_id=None, options=None):
        self._h = None
        L = C.lib()
        h = ctypes.c_void_p()
        C.check(L.amg_create(int(device), int(rank), int(nranks), nccl_id, ctypes.byref(h)), "amg_create")
        self._h = h
        self.device = device
        self.levels = []
        self.n_levels = 0
        for k, v in (options or {}).items():
            C.check(L.amg_set_option(self._h, k.encode(), int(v)), f"option {k}")

    # ------------------------------------------------------------------ upload
    @classmethod
    def from_reference(cls, h, device=0, options=None):
        """Upload a reference hierarchy (``AmgHierarchy`` or ``HostHierarchy``)."""
        dh = cls(device=device, options=options)
        dh._upload(h)
        return dh

    @classmethod
    def from_matrices(cls, mats, device=0, options=None):
        """Matrix container (no hierarchy): matrix i becomes ``matrix(i, "a")``.

        Used for standalone SpMV parity on arbitrary (ragged, rectangular)
        CSR matrices; the solve entry points reject such a handle.
        """
        dh = cls(device=device, options=options)
        L = C.lib()
        C.check(L.amg_set_levels(dh._h, len(mats)), "amg_set_levels")
        dh.n_levels = len(mats)
        dh.levels = []
        for k, m in enumerate(mats):
            info = {"n": int(m.nrows), "nnz": {}}
            dh._put(k, "a", m, info)
            dh.levels.append(info)
        C.check(L.amg_finalize(dh._h), "amg_finalize")
        return dh

    @classmethod
    def from_plan(cls, plan, device=0, nccl_id=None, options=None):
        """Upload one rank's share of a partitioned hierarchy (``partition.plan_hierarchy``).

        ``nccl_id``: the 128-byte id from :func:`nccl_unique_id` on rank 0,
        shared with every rank; one process per GPU.
        """
        import ctypes as ct

        idbuf = None
        if plan.nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise AmgError("from_plan: nranks > 1 needs the 128-byte NCCL unique id")
            idbuf = ct.create_string_buffer(bytes(nccl_id), 128)
        dh = cls(device=device, rank=plan.rank, nranks=plan.nranks, nccl_id=idbuf, options=options)
        L = C.lib()
        nl = len(plan.starts)
        C.check(L.amg_set_levels(dh._h, nl), "amg_set_levels")
        dh.n_levels = nl
        dh.levels = []
        if plan.nranks > 1:
            for k in range(nl):
                s = np.ascontiguousarray(plan.starts[k], dtype=np.int64)
                C.check(L.amg_set_partition(dh._h, k, C.ptr(s)), "amg_set_partition")
            C.check(L.amg_set_agglomeration(dh._h, int(min(plan.agglom_level, nl - 1))), "amg_set_agglomeration")
        for k in range(nl):
            info = {"n": plan.n_local(k) if plan.nranks > 1 else int(plan.mats[(k, "a")].csr.nrows), "nnz": {}}
            for slot in ("a", "p", "pt", "g", "gt"):
                lm = plan.mats.get((k, slot))
                if lm is None:
                    continue
                dh._put(k, slot, lm.csr, info)
                hp = lm.halo
                if hp is not None and plan.nranks > 1:
                    rp = np.asarray(hp.recv_peers, dtype=np.int32)
                    rc = np.asarray(hp.recv_counts, dtype=np.int64)
                    sp = np.asarray(hp.send_peers, dtype=np.int32)
                    sc = np.asarray([i.size for i in hp.send_idx], dtype=np.int64)
                    si = (np.concatenate(hp.send_idx) if hp.send_idx else np.zeros(0)).astype(np.int32)
                    C.check(L.amg_set_halo(dh._h, k, C.SLOT[slot], hp.n_own, hp.n_halo, rp.size, C.ptr(rp), C.ptr(rc),
                                           sp.size, C.ptr(sp), C.ptr(sc), C.ptr(si)), f"halo L{k}.{slot}")
                    info.setdefault("n_own", {})[slot] = hp.n_own
            if k in plan.smoothers:
                kind, omega, inv = plan.smoothers[k]
                if kind == "jacobi":
                    inv = _host_f64(inv)
                    C.check(L.amg_set_smoother(dh._h, k, C.AMG_SMOOTHER_JACOBI, omega, C.ptr(inv), inv.size), "smoother")
                else:
                    C.check(L.amg_set_smoother(dh._h, k, C.AMG_SMOOTHER_FSAI, omega, None, 0), "smoother")
            dh.levels.append(info)
        dh._upload_coarse(plan.factor_kind, plan.factor)
        C.check(L.amg_set_cycle(dh._h, plan.nu1, plan.nu2), "amg_set_cycle")
        dh.nu1, dh.nu2 = plan.nu1, plan.nu2
        C.check(L.amg_finalize(dh._h), "amg_finalize")
        dh.A0 = dh.matrix(0, "a")
        dh.vcycle = DeviceVcycle(dh)
        return dh

    def _upload_coarse(self, kind, factor):
        L = C.lib()
        if kind in ("cholesky", "cholesky+shift"):
            c, lower = factor
            if not lower:
                raise AmgError("expected a lower Cholesky factor (hierarchy.py:127)")
            c = np.ascontiguousarray(np.tril(c), dtype=np.float64)
            C.check(L.amg_upload_coarse(self._h, c.shape[0], C.ptr(c), C.AMG_COARSE_CHOLESKY, None), "amg_upload_coarse")
        else:
            lu, piv = factor
            lu = np.ascontiguousarray(lu, dtype=np.float64)
            piv = np.ascontiguousarray(piv, dtype=np.int32)
            C.check(L.amg_upload_coarse(self._h, lu.shape[0], C.ptr(lu), C.AMG_COARSE_LU, C.ptr(piv)), "amg_upload_coarse")
        self.factor_kind = kind
        self.nc = int(np.asarray(factor[0]).shape[0])

    def _upload(self, h):
        L = C.lib()
        levels = h.levels
        nl = len(levels)
        C.check(L.amg_set_levels(self._h, nl), "amg_set_levels")
        self.n_levels = nl
        self.levels = []
        for k, lvl in enumerate(levels):
            info = {"n": int(lvl.a.nrows), "nnz": {}}
            self._put(k, "a", lvl.a, info)
            if k < nl - 1:
                self._put(k, "p", lvl.p, info)
                self._put(k, "pt", lvl.pt, info)
                sm = lvl.smoother
                if sm.kind == "jacobi":
                    inv = _host_f64(sm.inv_diag)
                    C.check(L.amg_set_smoother(self._h, k, C.AMG_SMOOTHER_JACOBI, float(sm.omega), C.ptr(inv), inv.size),
                            "amg_set_smoother")
                else:
                    self._put(k, "g", sm.gmat, info)
                    self._put(k, "gt", sm.gmat_t, info)
                    C.check(L.amg_set_smoother(self._h, k, C.AMG_SMOOTHER_FSAI, float(sm.omega), None, 0),
                            "amg_set_smoother")
                info["omega"] = float(sm.omega)
                info["smoother"] = sm.kind
            self.levels.append(info)
        self._upload_coarse(h.factor_kind, h.factor)
        C.check(L.amg_set_cycle(self._h, int(h.config.nu1), int(h.config.nu2)), "amg_set_cycle")
        self.nu1, self.nu2 = int(h.config.nu1), int(h.config.nu2)
        C.check(L.amg_finalize(self._h), "amg_finalize")
        self.A0 = self.matrix(0, "a")
        self.vcycle = DeviceVcycle(self)

    def _put(self, k, slot, m, info):
        off = np.ascontiguousarray(m.row_offsets, dtype=np.int64)
        col = np.ascontiguousarray(m.col_indices, dtype=np.int32)
        val = np.ascontiguousarray(m.values, dtype=np.float64)
        C.check(C.lib().amg_upload_matrix(self._h, k, C.SLOT[slot], int(m.nrows), int(m.ncols),
                                          C.ptr(off), C.ptr(col), C.ptr(val)), f"upload L{k}.{slot}")
        info.setdefault("shape", {})[slot] = (int(m.nrows), int(m.ncols))
        info["nnz"][slot] = int(m.nnz)

    def matrix(self, level, slot):
        nr, nc = self.levels[level]["shape"][slot]
        return DeviceMatrix(self, level, slot, nr, nc, self.levels[level]["nnz"][slot])

    # ------------------------------------------------------------------ ops
    def _vec_in(self, x, n, op, shape):
        if _is_cuda_tensor(x):
            import torch

            if x.dtype != torch.float64 or not x.is_contiguous() or x.dim() != 1:
                raise AmgError(f"{op}: device vectors must be contiguous 1-D float64 tensors")
            if x.shape[0] != n:
                raise DimensionMismatchError(op, shape, tuple(x.shape))
            return x, 1
        if hasattr(x, "is_pinned") and x.is_pinned():  # pinned host tensor: async H2D / D2H
            import torch

            if x.dtype != torch.float64 or not x.is_contiguous() or x.dim() != 1:
                raise AmgError(f"{op}: pinned host vectors must be contiguous 1-D float64 tensors")
            if x.shape[0] != n:
                raise DimensionMismatchError(op, shape, tuple(x.shape))
            return x, 0
        a = _host_f64(x)
        if a.ndim != 1:
            raise AmgError(f"{op}: only 1-D vectors are supported on the device path")
        if a.shape[0] != n:
            raise DimensionMismatchError(op, shape, a.shape)
        return a, 0

    def _vec_in_like(self, x, n, op, shape, dev, like):
        """A second input vector (x0) staged to the residency of the first (b): the C
        side copies every vector of one call with one memcpy kind."""
        v, d = self._vec_in(x, n, op, shape)
        if d == dev:
            if dev == 1 and v.device != like.device:
                v = v.to(like.device)
            return v
        if dev == 1:
            import torch

            return torch.as_tensor(np.asarray(v.numpy() if hasattr(v, "numpy") else v, dtype=np.float64),
                                   device=like.device).contiguous()
        return np.ascontiguousarray(v.detach().cpu().numpy(), dtype=np.float64)

    def _vec_out(self, like, n):
        if _is_cuda_tensor(like):
            import torch

            return torch.empty(n, dtype=torch.float64, device=like.device)
        if hasattr(like, "is_pinned") and like.is_pinned():
            import torch

            return torch.empty(n, dtype=torch.float64, pin_memory=True)
        return np.empty(n, dtype=np.float64)

    def spmv(self, level, slot, x):
        """``spmv(A, x)`` (``amgkit/sparse.py:203-217``) for an uploaded matrix."""
        nr, nc = self.levels[level]["shape"][slot]
        nc = self.levels[level].get("n_own", {}).get(slot, nc)
        xin, dev = self._vec_in(x, nc, "spmv", (nr, nc))
        y = self._vec_out(xin, nr)
        C.check(C.lib().amg_spmv(self._h, level, C.SLOT[slot], C.ptr(xin), C.ptr(y), dev), "spmv")
        return y

    def apply_smoother(self, level, b, x0, steps):
        """``apply_smoother(sm_k, A_k, b, x0, steps)`` (``amgkit/smoothers.py:168-173``)."""
        n = self.levels[level]["n"]
        bin_, dev = self._vec_in(b, n, "apply_smoother", (n, n))
        x0in = None
        if x0 is not None:
            x0in = self._vec_in_like(x0, n, "apply_smoother", (n, n), dev, bin_)
        x = self._vec_out(bin_, n)
        C.check(C.lib().amg_smoother(self._h, level, C.ptr(bin_), C.ptr(x0in), C.ptr(x), int(steps), dev),
                "apply_smoother")
        return x

    def coarse_solve(self, y):
        """``AmgHierarchy.coarse_solve`` (``amgkit/hierarchy.py:149-152``)."""
        yin, dev = self._vec_in(y, self.nc, "coarse_solve", (self.nc, self.nc))
        z = self._vec_out(yin, self.nc)
        C.check(C.lib().amg_coarse_solve(self._h, C.ptr(yin), C.ptr(z), dev), "coarse_solve")
        return z

    def smoother(self, level):
        """The level's smoother as an object (``amgkit.smoothers.Smoother``'s role in
        ``apply_smoother(sm, A, b, x0, steps)``); the device owns the factors."""
        return DeviceSmoother(self, int(level))

    def apply_vcycle(self, y, level=0):
        """``vcycle(h, y, level)`` (``amgkit/hierarchy.py:294-312``)."""
        n = self.levels[level]["n"]
        yin, dev = self._vec_in(y, n, "vcycle", (n, n))
        z = self._vec_out(yin, n)
        if level == 0:
            C.check(C.lib().amg_vcycle(self._h, C.ptr(yin), C.ptr(z), dev), "vcycle")
        else:
            C.check(C.lib().amg_vcycle_level(self._h, int(level), C.ptr(yin), C.ptr(z), dev), "vcycle")
        return z

    def time_spmv(self, level, slot, reps=20):
        """Average device ms of one SpMV launch (CUDA events on the library stream)."""
        ms = C.D(0.0)
        which = 5 if slot == "smooth" else C.SLOT[slot]  # "smooth": one smoother step from zero
        C.check(C.lib().amg_time_spmv(self._h, level, which, int(reps), ctypes.byref(ms)), "time_spmv")
        return ms.value

    def set_option(self, key, value):
        C.check(C.lib().amg_set_option(self._h, key.encode(), int(value)), f"option {key}")

    LAYOUTS = ("csr", "padded", "pattern", "sell", "sell_pattern", "symd", "leaves", "empty", "sell_uniform", "sell_sorted", "split", "dict", "wcsr")
    _SLOTS = {"a": 0, "p": 1, "pt": 2, "g": 3, "gt": 4}

    def layout(self, level, slot):
        """Name of the device layout matrix `slot` of `level` runs on (diagnostics)."""
        v = ctypes.c_int32(0)
        C.check(C.lib().amg_matrix_layout(self._h, int(level), self._SLOTS[slot], ctypes.byref(v)), "amg_matrix_layout")
        return self.LAYOUTS[v.value]

    def matrix_bytes(self, level, slot):
        """(stored, vectors): bytes one SpMV launch of this matrix's layout must move
        (``amg_matrix_bytes``; the roofline numerator of the chosen layout)."""
        st, ve = ctypes.c_int64(0), ctypes.c_int64(0)
        C.check(C.lib().amg_matrix_bytes(self._h, int(level), self._SLOTS[slot], ctypes.byref(st), ctypes.byref(ve)),
                "amg_matrix_bytes")
        return int(st.value), int(ve.value)

    def stats(self):
        s = C.Stats()
        C.check(C.lib().amg_get_stats(self._h, ctypes.byref(s)), "amg_get_stats")
        return {f: getattr(s, f) for f, _ in C.Stats._fields_}

    def close(self):
        if self._h is not None and self._h.value:
            C.lib().amg_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def layout_bytes_per_iter(dh, h):
    """Bytes per PCG iteration on the layouts the device actually runs.

    Same application counts and vector terms as :func:`model_bytes_flops`,
    but each matrix application costs the bytes its chosen layout must stream
    (``DeviceHierarchy.matrix_bytes``: e.g. the symmetric stencil layout
    stores only the diagonals d >= 0, uniform SELL skips no slots) instead of
    the 12 B/entry CSR model.  The roofline fraction on these bytes cannot
    exceed 1 unless the hardware moved fewer bytes than the data structure
    holds (L2 reuse across kernels).
    """
    levels = h.levels
    nu1, nu2 = int(h.config.nu1), int(h.config.nu2)

    def M(k, slot):
        return dh.matrix_bytes(k, slot)[0]

    nbytes = 0
    for k in range(len(levels) - 1):
        lv = levels[k]
        n_k, n_c = lv.a.nrows, levels[k + 1].a.nrows
        n_a = (max(nu1 - 1, 0) + 1 + nu2) if nu1 else nu2
        steps = nu1 + nu2
        nbytes += n_a * M(k, "a") + M(k, "p") + M(k, "pt")
        if lv.smoother.kind == "fsai":
            nbytes += steps * (M(k, "g") + M(k, "gt"))
        else:
            nbytes += steps * 8 * 3 * n_k
        nbytes += 8 * (18 * n_k + 2 * n_c)
    nL = levels[-1].a.nrows
    nbytes += 8 * nL * (nL + 1) + 16 * nL
    n0 = levels[0].a.nrows
    nbytes += M(0, "a") + 8 * 13 * n0
    return int(nbytes)


def model_bytes_flops(h):
    """Algorithmic bytes and flops per PCG iteration (SURVEY.md 8(d) model).

    M(X) = 12 nnz(X) + 4 (rows(X) + 1) per application; per level k < L with
    nu1 = nu2 = 1 and FSAI: 2 M(A_k) + 4 M(G_k) + M(P_k) + M(P_k^T) +
    8 (18 n_k + 2 n_{k+1}); coarsest 8 n_L (n_L + 1) + 16 n_L; outside the
    V-cycle M(A_0) + 8 * 13 n_0.  General nu1 / nu2 and Jacobi count the
    applications actually performed (the first pre-smoothing step skips A.0).
    Flops: 2 per stored entry per application, 2 n_L^2 for the dense solve,
    12 n_0 for the PCG vector updates.
    """
    def M(m):
        return 12 * m.nnz + 4 * (m.nrows + 1)

    levels = h.levels
    nu1, nu2 = int(h.config.nu1), int(h.config.nu2)
    nbytes = 0
    flops = 0
    for k in range(len(levels) - 1):
        lv = levels[k]
        n_k, n_c = lv.a.nrows, levels[k + 1].a.nrows
        n_a = max(nu1 - 1, 0) + 1 + nu2  # residual spmv count (pre steps after the first, cgc, post)
        if nu1 == 0:
            n_a = nu2
        steps = nu1 + nu2
        nbytes += n_a * M(lv.a) + M(lv.p) + M(lv.pt)
        flops += 2 * n_a * lv.a.nnz + 2 * lv.p.nnz + 2 * lv.pt.nnz
        if lv.smoother.kind == "fsai":
            nbytes += 2 * steps * M(lv.smoother.gmat)
            flops += 4 * steps * lv.smoother.gmat.nnz
        else:
            nbytes += steps * 8 * 3 * n_k
            flops += 3 * steps * n_k
        nbytes += 8 * (18 * n_k + 2 * n_c)
    nL = levels[-1].a.nrows
    nbytes += 8 * nL * (nL + 1) + 16 * nL
    flops += 2 * nL * nL
    n0 = levels[0].a.nrows
    nbytes += M(levels[0].a) + 8 * 13 * n0
    flops += 2 * levels[0].a.nnz + 12 * n0
    return int(nbytes), int(flops)
