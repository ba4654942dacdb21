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


class DistOracle:
    def __init__(self, plan, dist):
        self.plan = plan
        self.dist = dist
        self.nl = len(plan.starts)

    # ---------------------------------------------------------------- comm
    def exchange(self, lm, x_own):
        import torch

        halo = lm.halo
        x_ext = np.empty(halo.n_own + halo.n_halo)
        x_ext[: halo.n_own] = x_own
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
        for r in reqs:
            r.wait()
        pos = halo.n_own
        for buf in recv_bufs:
            x_ext[pos:pos + buf.numel()] = buf.numpy()
            pos += buf.numel()
        return x_ext

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
        lm = self.plan.mats[(k, slot)]
        x = self.exchange(lm, x_local) if lm.halo is not None else x_local
        return O.spmv(lm.csr, x)

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
