"""Multi-GPU plans on CPU: world_size 2 / 3 with the gloo backend.

The row-block partition (partition.py) is executed by the distributed
restatement (oracle/distributed.py) and compared with the single-process
oracle: every distributed SpMV row and every V-cycle must be bit-identical
(entries keep their reference order; the replicated coarse solve sees the
bit-identical all-gathered vector), PCG within +-1 iteration.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, agglom, out_q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from golden_io import load_case, matrices_of
    from oracle import solve as O
    from oracle.distributed import DistOracle
    from paper_2102_07417_b200.partition import plan_hierarchy

    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        c = load_case(case)
        h = c["h"]
        plan = plan_hierarchy(h, world, rank, agglom_rows=agglom)
        D = DistOracle(plan, dist)
        res = {"rank": rank, "ok": True, "msgs": []}
        # every distributed matrix (non-replicated levels): bitwise rows
        for k, slot, m in matrices_of(h):
            if k >= plan.agglom_level:
                continue
            x = c["vec"][f"spmv_L{k}_{slot}_x"]
            lm = plan.mats[(k, slot)]
            cs = plan.starts[k + 1] if slot == "p" else plan.starts[k]
            if slot == "p" and k + 1 >= plan.agglom_level:
                xl = x
            else:
                xl = x[cs[rank]:cs[rank + 1]]
            y = D.spmv(k, slot, xl)
            ref = c["vec"][f"spmv_L{k}_{slot}_y"][lm.row0:lm.row0 + lm.csr.nrows]
            if not np.array_equal(y, ref):
                res["ok"] = False
                res["msgs"].append(f"spmv L{k}.{slot}")
        s0 = plan.starts[0]
        y = c["vec"]["y"]
        z = D.vcycle(y[s0[rank]:s0[rank + 1]])
        if not np.array_equal(z, O.vcycle(h, y)[s0[rank]:s0[rank + 1]]):
            res["ok"] = False
            res["msgs"].append("vcycle")
        if "pcg" in c["expect"]:
            b = c["vec"]["b"]
            x, its, relres, conv = D.pcg(b[s0[rank]:s0[rank + 1]])
            res["pcg"] = (its, relres, conv, x)
        res["agglom"] = plan.agglom_level
        res["split_spmvs"] = D.split_spmvs
        out_q.put(res)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        out_q.put({"rank": rank, "ok": False, "msgs": [traceback.format_exc()]})


def _run(case, world, agglom):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, agglom, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(outs, key=lambda d: d["rank"])


@pytest.mark.parametrize("case,world,agglom", [
    ("poisson7_12", 2, 0),        # only the coarsest level replicated
    ("poisson7_12", 2, 700),      # agglomerate from level 1
    ("hetero27_10", 3, 0),
    ("rtanis7_12", 2, 100),
    ("poisson2d_16_jacobi", 2, 0),
    ("elasticity_3_bamg", 2, 0),
])
def test_distributed_plan_matches_single_process(case, world, agglom):
    from golden_io import load_case

    outs = _run(case, world, agglom)
    for o in outs:
        assert o["ok"], o["msgs"]
    if case == "poisson7_12" and agglom == 0:  # level 0 blocks large enough for the overlap split
        assert all(o["split_spmvs"] > 0 for o in outs)
    c = load_case(case)
    if "pcg" in c["expect"]:
        exp = c["expect"]["pcg"]
        its = {o["pcg"][0] for o in outs}
        assert len(its) == 1  # every rank takes the same decisions
        it = its.pop()
        assert abs(it - exp["n_iterations"]) <= 1
        assert all(o["pcg"][2] for o in outs)
        x = np.concatenate([o["pcg"][3] for o in outs])
        b = c["vec"]["b"]
        from oracle import solve as O

        rel = np.linalg.norm(b - O.spmv(c["h"].levels[0].a, x)) / np.linalg.norm(b)
        assert rel <= exp["rtol"] * 1.0001


def test_interior_range_matches_brute_force():
    # the overlap split (partition.interior_range == csrc interior_range): rows
    # inside [lo, hi) never touch a halo column, lo / hi are 128-aligned
    from golden_io import load_case
    from paper_2102_07417_b200.partition import interior_range, plan_hierarchy

    h = load_case("hetero27_10")["h"]
    seen = 0
    for world in (2, 3):
        for r in range(world):
            plan = plan_hierarchy(h, world, r, agglom_rows=0)
            for key, lm in plan.mats.items():
                if lm.halo is None:
                    continue
                lo, hi = interior_range(lm.csr, lm.halo.n_own)
                assert lo % 128 == 0 and hi % 128 == 0 and lo <= hi
                o = np.asarray(lm.csr.row_offsets)
                for row in range(lo, hi):
                    assert np.all(lm.csr.col_indices[o[row]:o[row + 1]] < lm.halo.n_own)
                seen += hi > lo
    assert seen > 0


def test_partition_inherits_contiguous_ownership():
    from golden_io import load_case
    from paper_2102_07417_b200.partition import partition_rows, plan_hierarchy

    h = load_case("poisson7_12")["h"]
    plan = plan_hierarchy(h, 4, 1, agglom_rows=0)
    for s in plan.starts:
        assert s[0] == 0 and np.all(np.diff(s) >= 0)
    assert np.array_equal(partition_rows(10, 3), [0, 4, 7, 10])
    # halo plans are consistent: what rank r sends to q is what q receives from r
    plans = [plan_hierarchy(h, 3, r, agglom_rows=0) for r in range(3)]
    for key, lm in plans[0].mats.items():
        if lm.halo is None:
            continue
        for r in range(3):
            hr = plans[r].mats[key].halo
            for q, idx in zip(hr.send_peers, hr.send_idx):
                hq = plans[q].mats[key].halo
                seg = hq.recv_peers.index(r)
                off = sum(hq.recv_counts[:seg])
                got = hq.halo_cols[off:off + hq.recv_counts[seg]]
                c0 = plans[r].starts[key[0] + 1 if key[1] == "p" else key[0]][r]
                assert np.array_equal(got, idx.astype(np.int64) + c0)
