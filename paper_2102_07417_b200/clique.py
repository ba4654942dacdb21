"""Single-process multi-GPU clique: N GPUs driven from one host process.

The reference's caller is single-process (``amgkit/cli.py:257-274``:
``pcg(lambda v: spmv(A0, v), b, apply_m=lambda r: vcycle(h, r))``).  A
:class:`DeviceClique` gives that caller N GPUs without torch.distributed: it
plans the row partition of every level once (``partition.plan_hierarchy``,
the DSMat stripes of ``amgkit/striped.py:28-106`` mapped to GPUs), creates
one library handle per GPU (one NCCL rank each, communicator initialised
collectively from N host threads), and runs every solve on all GPUs at once
-- one host thread per GPU inside ``amg_pcg`` (ctypes releases the GIL), each
on its slice of b -- then gathers x.  Results equal the one-process-per-GPU
path bit for bit (same plans, same kernels, same collectives).

    cl = DeviceClique(h, devices=[0, 1, 2, 3])
    res = pcg(cl.A0, b, apply_m=cl.vcycle, config=KrylovConfig(rtol=1e-8))

With one device it is a thin wrapper around a single-GPU handle.
"""
from __future__ import annotations

import threading

import numpy as np

from .device import DeviceHierarchy, nccl_unique_id
from .errors import AmgError

__all__ = ["DeviceClique"]


class _CliqueOp:
    """``cl.A0`` / ``cl.vcycle``: the operator callables of the reference protocol."""

    def __init__(self, clique, kind):
        self.clique = clique
        self.kind = kind

    def __call__(self, v):
        return self.clique.spmv_a0(v) if self.kind == "A0" else self.clique.apply_vcycle(v)


def _run_all(fns):
    """Run fns[i]() on N threads; re-raise the first failure."""
    out = [None] * len(fns)
    err = [None] * len(fns)

    def work(i):
        try:
            out[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[i] = e

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


class DeviceClique:
    """One hierarchy row-partitioned over ``devices`` (one handle per GPU)."""

    def __init__(self, h, devices, agglom_rows=50000, options=None):
        from .partition import plan_hierarchy

        self.devices = [int(d) for d in devices]
        if not self.devices:
            raise AmgError("DeviceClique: no devices")
        n = len(self.devices)
        self.n0 = int(h.levels[0].a.nrows)
        plans = [plan_hierarchy(h, n, r, agglom_rows=agglom_rows) for r in range(n)]
        self.starts = np.asarray(plans[0].starts[0], dtype=np.int64)
        uid = nccl_unique_id() if n > 1 else None
        # NCCL communicator creation is collective: every rank's handle at once
        self.ranks = _run_all([
            (lambda r=r: DeviceHierarchy.from_plan(plans[r], device=self.devices[r], nccl_id=uid, options=options))
            for r in range(n)
        ])
        self.A0 = _CliqueOp(self, "A0")
        self.vcycle = _CliqueOp(self, "vcycle")

    @property
    def nranks(self):
        return len(self.ranks)

    def scatter(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.shape != (self.n0,):
            from .errors import DimensionMismatchError

            raise DimensionMismatchError("clique", (self.n0,), v.shape)
        return [v[self.starts[r]:self.starts[r + 1]] for r in range(self.nranks)]

    def gather(self, parts):
        return np.concatenate([np.asarray(p) for p in parts])

    def pcg(self, b, x0=None, config=None):
        from .krylov import KrylovResult, pcg

        bs = self.scatter(b)
        xs = self.scatter(x0) if x0 is not None else [None] * self.nranks
        res = _run_all([
            (lambda r=r: pcg(self.ranks[r].A0, bs[r], apply_m=self.ranks[r].vcycle, x0=xs[r], config=config))
            for r in range(self.nranks)
        ])
        r0 = res[0]
        return KrylovResult(x=self.gather([r.x for r in res]), converged=r0.converged, n_iterations=r0.n_iterations,
                            relres=r0.relres, history=r0.history, restarts=0,
                            solve_ms=max(r.solve_ms for r in res))

    def apply_vcycle(self, y):
        ys = self.scatter(y)
        zs = _run_all([(lambda r=r: self.ranks[r].vcycle(ys[r])) for r in range(self.nranks)])
        return self.gather(zs)

    def spmv_a0(self, x):
        xs = self.scatter(x)
        ys = _run_all([(lambda r=r: self.ranks[r].A0(xs[r])) for r in range(self.nranks)])
        return self.gather(ys)

    def close(self):
        for d in self.ranks:
            d.close()
        self.ranks = []
