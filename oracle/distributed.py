"""Distributed restatement of the solve path over a partition plan
(TEST INFRASTRUCTURE ONLY -- checks the multi-GPU plans on CPU with gloo).

Runs the reference algorithm (oracle/solve.py) rank by rank on the local
matrices of ``paper_2102_07417_b200.partition.plan_hierarchy``: halo
exchanges with torch.distributed point-to-point, the restricted vector
all-gathered at the agglomeration level, dots as per-rank partials combined
in rank order.  The device multi-GPU path executes exactly these plans with
NCCL; this emulator is what the gloo tests compare against the
single-process oracle.
"""
from __future__ import annotations

import numpy as np

from . import solve as O


def _rows(m, lo, hi):
    """Rows [lo, hi) of a CSR matrix (same column space)."""
    from paper_2102_07417_b200.problems import Csr

    o = np.asarray(m.row_offsets, dtype=np.int64)
    return Csr(hi - lo, m.ncols, o[lo:hi + 1] - o[lo], m.col_indices[o[lo]:o[hi]], m.values[o[lo]:o[hi]])


class DistOracle:
    def __init__(self, plan, dist):
        self.plan = plan
        self.dist = dist
        self.nl = len(plan.starts)
        self.split_spmvs = 0  # SpMVs that ran the interior / boundary split

    # ---------------------------------------------------------------- comm
    def exchange_begin(self, lm, x_own):
        """Post the halo receives / sends (non-blocking, as the device's comm stream)."""
        import torch

        halo = lm.halo
        reqs, recv_bufs = [], []
        for q, cnt in zip(halo.recv_peers, halo.recv_counts):
            buf = torch.empty(cnt, dtype=torch.float64)
            reqs.append(self.dist.irecv(buf, src=q))
            recv_bufs.append(buf)
        sends = []
        for q, idx in zip(halo.send_peers, halo.send_idx):
            t = torch.from_numpy(np.ascontiguousarray(x_own[idx]))
            sends.append(t)
            reqs.append(self.dist.isend(t, dst=q))
        return reqs, recv_bufs, sends

    def exchange_end(self, lm, x_ext, pending):
        reqs, recv_bufs, _ = pending
        for r in reqs:
            r.wait()
        pos = lm.halo.n_own
        for buf in recv_bufs:
            x_ext[pos:pos + buf.numel()] = buf.numpy()
            pos += buf.numel()
        return x_ext

    def exchange(self, lm, x_own):
        halo = lm.halo
        x_ext = np.empty(halo.n_own + halo.n_halo)
        x_ext[: halo.n_own] = x_own
        return self.exchange_end(lm, x_ext, self.exchange_begin(lm, x_own))

    def allgather_level(self, k, piece):
        import torch

        s = self.plan.starts[k]
        m = int(np.max(np.diff(s)))
        t = torch.zeros(m, dtype=torch.float64)
        t[: piece.size] = torch.from_numpy(piece)
        outs = [torch.zeros(m, dtype=torch.float64) for _ in range(self.plan.nranks)]
        self.dist.all_gather(outs, t)
        return np.concatenate([outs[q].numpy()[: s[q + 1] - s[q]] for q in range(self.plan.nranks)])

    def dot(self, a, b):
        import torch

        part = torch.tensor([float(a @ b)], dtype=torch.float64)
        outs = [torch.zeros(1, dtype=torch.float64) for _ in range(self.plan.nranks)]
        self.dist.all_gather(outs, part)
        tot = 0.0
        for o in outs:  # fixed rank order
            tot += float(o[0])
        return tot

    # ---------------------------------------------------------------- ops
    def spmv(self, k, slot, x_local):
        """The device's overlap schedule (csrc/capi.cu launch_spmv): interior rows
        from owned columns while the halo is in flight -- the halo segment holds
        NaN until it arrives, so an interior row reading it would show -- then
        the boundary rows [0, lo) + [hi, n)."""
        from paper_2102_07417_b200.partition import interior_range

        lm = self.plan.mats[(k, slot)]
        if lm.halo is None:
            return O.spmv(lm.csr, x_local)
        halo = lm.halo
        x_ext = np.full(halo.n_own + halo.n_halo, np.nan)
        x_ext[: halo.n_own] = x_local
        pending = self.exchange_begin(lm, x_local)
        lo, hi = interior_range(lm.csr, halo.n_own)
        y = np.empty(lm.csr.nrows)
        if hi > lo:
            y[lo:hi] = O.spmv(_rows(lm.csr, lo, hi), x_ext)
            self.split_spmvs += 1
        self.exchange_end(lm, x_ext, pending)
        if hi > lo:
            y[:lo] = O.spmv(_rows(lm.csr, 0, lo), x_ext)
            y[hi:] = O.spmv(_rows(lm.csr, hi, lm.csr.nrows), x_ext)
        else:
            y[:] = O.spmv(lm.csr, x_ext)
        return y

    def smooth(self, k, b, x0, steps):
        kind, omega, inv = self.plan.smoothers[k]
        x = np.array(x0, dtype=np.float64, copy=True)
        for _ in range(steps):
            r = b - self.spmv(k, "a", x)
            z = inv * r if kind == "jacobi" else self.spmv(k, "gt", self.spmv(k, "g", r))
            x += omega * z
        return x

    def coarse(self, y):
        class _H:
            pass

        h = _H()
        h.factor, h.factor_kind = self.plan.factor, self.plan.factor_kind
        return O.coarse_solve(h, y)

    def vcycle(self, y, k=0):
        p = self.plan
        if k == self.nl - 1:
            return self.coarse(y)
        x = self.smooth(k, y, np.zeros_like(y), p.nu1)
        r = y - self.spmv(k, "a", x)
        rc = self.spmv(k, "pt", r)
        if k + 1 == p.agglom_level:
            rc = self.allgather_level(k + 1, rc)
        dc = self.vcycle(rc, k + 1)
        x = x + self.spmv(k, "p", dc)
        return self.smooth(k, y, x, p.nu2)

    def pcg(self, b, rtol=1e-8, max_iters=5000, recompute_every=50):
        """krylov.py:40-92 control flow with distributed dots."""
        A = lambda v: self.spmv(0, "a", v)
        M = self.vcycle
        norm = lambda v: np.sqrt(self.dot(v, v))
        x = np.zeros_like(b)
        bnorm = norm(b)
        if bnorm == 0.0:
            return x, 0, 0.0, True
        r = b - A(x)
        z = M(r)
        p = z.copy()
        rz = self.dot(r, z)
        relres = norm(r) / bnorm
        if relres <= rtol:
            return x, 0, relres, True
        for it in range(1, max_iters + 1):
            q = A(p)
            curv = self.dot(p, q)
            if curv <= 0.0:
                raise O.NotSpdError(f"iteration {it}: direction with curvature {curv:.3e}")
            alpha = rz / curv
            x += alpha * p
            r -= alpha * q
            if it % recompute_every == 0:
                r = b - A(x)
            relres = norm(r) / bnorm
            if relres <= rtol:
                tr = b - A(x)
                relres = norm(tr) / bnorm
                if relres <= rtol:
                    return x, it, relres, True
                r = tr
            z = M(r)
            rz_new = self.dot(r, z)
            beta = rz_new / rz
            rz = rz_new
            p = z + beta * p
        return x, max_iters, relres, False
