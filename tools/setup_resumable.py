"""Resumable, per-level replay of the REFERENCE hierarchy setup (build container only).

``amgkit.setup`` (``/root/reference/pkg/src/amgkit/hierarchy.py:155-223``) builds
the whole hierarchy in one call; for the BASELINE configs 4-5 that is hours of
single-threaded Python.  This wrapper runs the SAME loop body --
the reference's own ``_build_smoother``, ``compute_soc`` / ``filter_soc``,
``pmis`` (seed ``coarsen_seed + depth``), ``_build_prolongation``,
``galerkin_product``, ``transpose``, ``restrict_testspace`` -- one level at a
time and pickles every finished level (plus the loop state: test space,
symmetry flag, warnings) into ``<state_dir>/level_<k>.pkl``.  A restarted run
loads the finished levels and continues with the next one, so an interrupted
setup loses at most one level.  The result is an ordinary ``AmgHierarchy``
(coarsest factor by the reference's ``AmgHierarchy.__init__``); it is
bit-identical to ``amgkit.setup`` on the same input (tests/test_hiercache.py).

Setup is not on the solve path; nothing here runs on the GPU box.
"""
from __future__ import annotations

import os
import pickle
import sys
import time

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)


def setup_resumable(A, config, state_dir, log=None):
    import numpy as np

    from amgkit import hierarchy as H

    cfg = config.validate()
    os.makedirs(state_dir, exist_ok=True)
    levels = [H.Level(a=A)]
    symmetric = H.is_symmetric(A)
    ts = None
    warnings = []
    done = False
    depth = 0
    # finished levels of an earlier run
    while os.path.exists(os.path.join(state_dir, f"level_{depth}.pkl")):
        with open(os.path.join(state_dir, f"level_{depth}.pkl"), "rb") as f:
            st = pickle.load(f)
        levels[-1] = st["level"]
        ts, symmetric, warnings, done = st["ts"], st["symmetric"], st["warnings"], st["done"]
        if st["next_a"] is not None:
            levels.append(H.Level(a=st["next_a"]))
        depth += 1
        if log:
            log(f"resumed level {depth - 1} ({levels[-1].a.nrows} rows next)")
        if done:
            break
    while not done and depth < cfg.max_levels - 1:
        t0 = time.perf_counter()
        lvl = levels[-1]
        a = lvl.a
        n = a.nrows
        next_a = None
        if n <= cfg.max_coarse:
            done = True
        else:
            # hierarchy.py:170-219, one iteration
            sm = H._build_smoother(a, cfg)
            lvl.smoother = sm
            if ts is None and H._needs_testspace(cfg):
                ts = H._initial_testspace(a, sm, cfg)
            lvl.testspace = ts
            g = H.compute_soc(a, cfg.soc_kind, vectors=ts.vectors if ts is not None else None)
            if cfg.soc_avg_degree is not None:
                H.filter_soc(g, avg_degree=cfg.soc_avg_degree)
            else:
                H.filter_soc(g, theta=cfg.soc_theta)
            cf = H.pmis(g, seed=cfg.coarsen_seed + depth)
            lvl.cf = cf
            lvl.soc_stats = {"kept_edges": g.n_kept, "coarse": cf.n_coarse}
            if cf.n_coarse == 0 or cf.n_coarse >= cfg.stall_fraction * n:
                warnings.append(f"level {depth}: coarsening stalled ({cf.n_coarse} of {n}); factorizing here")
                done = True
            else:
                prol = H._build_prolongation(a, g, cf, ts, cfg)
                if cfg.smooth_p:
                    prol = H.smooth_prolongation(a, prol, omega=None, power_iters=cfg.power_iters, seed=cfg.seed)
                w_coarse = ts.vectors[cf.coarse_nodes] if ts is not None else np.ones((cf.n_coarse, 1))
                p = prol.matrix
                if cfg.filter_target in ("prolongation", "both") and cfg.filter_rho < 1.0:
                    p = H.filter_with_compensation(p, w_coarse, cfg.filter_rho)
                next_a = H.galerkin_product(a, p, symmetrize=None if symmetric else False)
                if cfg.filter_target in ("operator", "both") and cfg.filter_rho < 1.0:
                    next_a = H.filter_with_compensation(next_a, w_coarse, cfg.filter_rho)
                    symmetric = symmetric and H.is_symmetric(next_a)
                lvl.p = p
                lvl.pt = H.transpose(p)
                if ts is not None:
                    ts = H.restrict_testspace(ts, cf)
        tmp = os.path.join(state_dir, f"level_{depth}.pkl.tmp")
        with open(tmp, "wb") as f:
            pickle.dump({"level": lvl, "ts": ts, "symmetric": symmetric, "warnings": warnings, "done": done,
                         "next_a": next_a}, f, protocol=5)
        os.replace(tmp, os.path.join(state_dir, f"level_{depth}.pkl"))
        if log:
            log(f"level {depth}: {n} rows, {time.perf_counter() - t0:.1f} s")
        if next_a is not None:
            levels.append(H.Level(a=next_a))
        depth += 1
        if done:
            break
    h = H.AmgHierarchy(levels, cfg, symmetric=symmetric)
    h.setup_warnings = warnings
    return h
