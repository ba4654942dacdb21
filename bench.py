#!/usr/bin/env python
"""PCG + AMG solve-phase benchmark (BASELINE.json metric: solve ms/iter,
GFLOP/s and HBM-roofline fraction on B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl amgb200|reference]

Workload (``config.workload``): the largest single-GPU BASELINE configuration
whose reference setup could be run -- configs[3], anisotropic 3-D Poisson,
7-point stencil on 256^3 (16,777,216 unknowns, 117,047,296 nnz), eps = 1e-3 in
z, rhs uniform(-1,1) seed 42, classical AMG + FSAI from the reference's setup
(frozen in hier_cache/), PCG to rtol 1e-8.  ``--config`` runs
configs 1-3 (c1_poisson7_64, c2_hetero27_128, c3_elasticity_64) the same way.  A step = one complete PCG solve from x0 = 0 (initial
residual, every iteration, final true residual) with b already resident in
HBM; ``value`` = device time of the K solves / total iterations (ms per PCG
iteration; lower is better).  ``e2e`` = the same through the public API with
pinned host b / x (H2D + D2H inside the timed region).

``--impl reference``: the reference's solve path on the host CPU (the numpy
oracle that restates it bit for bit; the reference package itself cannot
travel to the GPU box), same hierarchy and RHS; a step = one PCG iteration.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

DEFAULT_CONFIG = "c4_rtanis7_256"
METRIC = "PCG+AMG solve ms/iter (GFLOP/s, HBM-roofline fraction alongside)"
WORKLOADS = {
    "c1_poisson7_64": "config 1: 3-D Poisson 7-pt 64^3 (262,144 unknowns), FSAI + classical AMG, PCG 1e-8",
    "c2_hetero27_128": ("config 2: 3-D heterogeneous diffusion 27-pt 128^3 (2,097,152 unknowns, 55.7 M nnz), "
                        "lognormal sigma=2, FSAI + classical AMG, PCG 1e-8"),
    "c3_elasticity_64": ("config 3: 3-D linear elasticity Q1 hexahedra 64^3 elements (811,200 dofs, 63.7 M nnz), "
                         "lognormal E sigma=1, FSAI + BAMG + rigid-body modes, PCG 1e-8"),
    "c4_rtanis7_256": ("config 4: anisotropic 3-D Poisson 7-pt 256^3 eps=1e-3 in z (16,777,216 unknowns, 117.0 M nnz), "
                       "FSAI + classical AMG, PCG 1e-8"),
    "t_rtanis7_256x64": "stand-in: config 4's x-y planes, 64 of its 256 planes (4,194,304 unknowns)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="amgb200", choices=("amgb200", "reference"))
    ap.add_argument("--config", default=os.environ.get("AMGB200_BENCH_CONFIG", DEFAULT_CONFIG))
    ap.add_argument("--cache", default=os.path.join(ROOT, "hier_cache"))
    ap.add_argument("--cpu-iters", type=int, default=2, help="PCG iterations in the cpu_baseline sample")
    ap.add_argument("--cpu-budget", type=float, default=150.0,
                    help="--impl reference: stop the W + K iteration sample after this many seconds")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of the row partition")
    ap.add_argument("--agglom-rows", type=int, default=50000, help="levels with <= this many rows are replicated")
    ap.add_argument("--partitioned", action="store_true", help="use the partition-plan upload even at N=1")
    ap.add_argument("--watchdog", type=float, default=900.0, help="abort (exit 3) if the GPU phase exceeds this")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.hd = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hd, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.hd, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.hd))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def report(self):
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config, layout=None, matrix=None):
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any
    (only when the summary was captured on the same matrix and device layout)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f).get(config, {})
        if layout is not None and d.get("layout") not in (None, layout):
            return None
        if matrix is not None and d.get("matrix", "L0.a") != matrix:
            return None
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def load(args):
    from paper_2102_07417_b200 import hiercache, problems

    d = os.path.join(args.cache, args.config)
    if not os.path.exists(os.path.join(d, "manifest.json")):
        raise SystemExit(f"bench: hierarchy cache {d} missing (run tools/export_hierarchy.py {args.config})")
    h = hiercache.load_hierarchy(d, verify=True)
    b = problems.build_rhs(args.config, h.levels[0].a.nrows)
    return h, b


def cpu_sample(h, b, iters, budget_s=None):
    """The oracle (reference restatement) on the host: ms of each of up to `iters` PCG
    iterations, stopping early once `budget_s` seconds of iterations have run."""
    from oracle import solve as O

    a0 = h.levels[0].a
    marks = []
    O.pcg(lambda v: O.spmv(a0, v), b, apply_m=lambda r: O.vcycle(h, r),
          config=O.KrylovConfig(rtol=1e-8), max_steps=iters, iter_marks=marks, time_budget=budget_s)
    dt = np.diff(marks) * 1e3
    return [float(x) for x in dt]


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    h, b = load(args)
    # bounded sample: W + K PCG iterations, cut at --cpu-budget seconds (config 4's
    # reference iteration alone takes ~17 s on one core); at least one warm-up
    # iteration and one timed iteration always run
    dts = cpu_sample(h, b, args.warmup + args.steps, budget_s=args.cpu_budget)
    warm = min(args.warmup, len(dts) - 1) if len(dts) > 1 else 0
    timed = dts[warm:warm + args.steps]
    steps = len(timed)
    ms = float(np.mean(timed))
    line = {
        "impl": "reference",
        "metric": METRIC, "value": ms, "unit": "ms/iter", "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator + reference setup hierarchy)",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "name": args.config,
                   "step": "one PCG iteration (SpMV A0, V-cycle, 3 dots, 3 axpys) of the reference path",
                   "requested_steps": args.steps, "requested_warmup": args.warmup,
                   "cpu_budget_s": args.cpu_budget},
        "cpu_baseline": {"value": ms, "unit": "ms/iter", "cores": 1, "kind": "port",
                         "sample": f"{steps} PCG iterations after {warm} warm-up iterations (W + K iterations "
                                   f"requested, cut at {args.cpu_budget:.0f} s), numpy oracle (bit-identical "
                                   "restatement of amgkit's solve path; numpy's kernels are single-threaded)"},
        "e2e": {"value": ms, "unit": "ms/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_cpu": _cpu_model(),
    }
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_amgb200(args):
    import torch

    import paper_2102_07417_b200 as amg
    from paper_2102_07417_b200.device import layout_bytes_per_iter, model_bytes_flops

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
    torch.cuda.set_device(local)
    h, b_host = load(args)
    n = b_host.size

    def _watchdog():
        time.sleep(args.watchdog)
        print(json.dumps({"error": f"bench watchdog: GPU phase exceeded {args.watchdog} s (rank {rank})"}), flush=True)
        os._exit(3)

    threading.Thread(target=_watchdog, daemon=True).start()
    partitioned = (world > 1 and not args.replicas) or args.partitioned
    if partitioned:
        from paper_2102_07417_b200.partition import plan_hierarchy

        plan = plan_hierarchy(h, world, rank, agglom_rows=args.agglom_rows)
        uid = None
        if world > 1:
            t = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
            if rank == 0:
                t.copy_(torch.tensor(list(amg.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(t, 0)
            uid = bytes(t.cpu().tolist())
        dh = amg.DeviceHierarchy.from_plan(plan, device=local, nccl_id=uid)
        s0 = plan.starts[0]
        lo, hi = (int(s0[rank]), int(s0[rank + 1])) if world > 1 else (0, n)
    else:
        plan = None
        dh = amg.DeviceHierarchy.from_reference(h, device=local)
        lo, hi = 0, n
    b_local = np.ascontiguousarray(b_host[lo:hi])
    b_dev = torch.tensor(b_local, device=f"cuda:{local}")
    cfg = amg.KrylovConfig(rtol=1e-8, max_iters=5000)
    bytes_iter, flops_iter = model_bytes_flops(h)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        res = amg.pcg(dh.A0, b_dev, apply_m=dh.vcycle, config=cfg)
    barrier()
    solve_ms, iters, launches = [], [], 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res = amg.pcg(dh.A0, b_dev, apply_m=dh.vcycle, config=cfg)
            st = dh.stats()
            solve_ms.append(st["solve_ms"])
            iters.append(res.n_iterations)
            launches += st["launches_last"]
    barrier()
    tot_ms = float(sum(solve_ms))
    tot_it = int(sum(iters))
    ms_iter = tot_ms / max(tot_it, 1)
    if dist is not None:
        t = torch.tensor([ms_iter], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_iter = float(t.item())
    # parity record of this run
    from oracle import solve as O  # checker only: true residual of the device answer
    x = res.x.cpu().numpy()
    if world > 1 and partitioned:
        m = int(max(np.diff(plan.starts[0])))
        tx = torch.zeros(m, dtype=torch.float64, device=f"cuda:{local}")
        tx[: x.size] = torch.from_numpy(x)
        outs = [torch.zeros(m, dtype=torch.float64, device=f"cuda:{local}") for _ in range(world)]
        dist.all_gather(outs, tx)
        s0 = plan.starts[0]
        x = np.concatenate([outs[q].cpu().numpy()[: s0[q + 1] - s0[q]] for q in range(world)])
    true_rel = float(np.linalg.norm(b_host - O.spmv(h.levels[0].a, x)) / np.linalg.norm(b_host))
    ref_its = h.meta.get("extra", {}).get("reference_solve", {}).get("n_iterations")

    # e2e: public API with pinned host buffers, copies inside the timed region
    # per call: wall time of pcg() (H2D of b, the solve, D2H of x, host control), median over the
    # steps (a Python / allocator hiccup on one call does not move it), garbage collector paused
    b_pin = torch.from_numpy(b_local).pin_memory()
    amg.pcg(dh.A0, b_pin, apply_m=dh.vcycle, config=cfg)
    barrier()
    gc.collect()
    gc.disable()
    e_per_iter = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r2 = amg.pcg(dh.A0, b_pin, apply_m=dh.vcycle, config=cfg)
        torch.cuda.synchronize()
        e_per_iter.append((time.perf_counter() - t0) * 1e3 / max(r2.n_iterations, 1))
    gc.enable()
    e2e_ms_iter = float(np.median(e_per_iter))
    e2e_mean = float(np.mean(e_per_iter))

    # dominant kernel: the SpMV with the largest share of a PCG iteration -- every matrix of the
    # levels above the cluster tail timed alone with CUDA events on the library stream
    # (amg_time_spmv), weighted by its applications per iteration (A: 2 per V-cycle + 1 outside
    # at level 0, G / G^T: 2, P / P^T: 1).  Roofline numerator = the bytes the chosen layout
    # must stream per launch (amg_matrix_bytes: stored values + indices + x once + y once).
    apps = {"a": 2, "g": 2, "gt": 2, "p": 1, "pt": 1}
    shares = []
    if plan is None:
        tail_level = dh.stats()["tail_level"]
        top = tail_level if tail_level > 0 else len(h.levels) - 1
        for k, lv in enumerate(h.levels[:max(top, 1)]):
            slots = ["a"]
            if lv.p is not None:
                slots += ["p", "pt"]
                if lv.smoother is not None and getattr(lv.smoother, "gmat", None) is not None:
                    slots += ["g", "gt"]
            for slot in slots:
                try:
                    t_ms = dh.time_spmv(k, slot, reps=10)
                except Exception:
                    continue
                n_app = apps[slot] + (1 if (k == 0 and slot == "a") else 0)
                shares.append((n_app * t_ms, k, slot, t_ms, n_app))
    if shares:
        shares.sort(reverse=True)
        _, dk, dslot, _, dn = shares[0]
    else:
        dk, dslot, dn = 0, "a", 3
    dm = (plan.mats[(dk, dslot)].csr if plan is not None else
          {"a": h.levels[dk].a, "p": h.levels[dk].p, "pt": h.levels[dk].pt,
           "g": getattr(h.levels[dk].smoother, "gmat", None), "gt": getattr(h.levels[dk].smoother, "gmat_t", None)}[dslot])
    k_ms = dh.time_spmv(dk, dslot, reps=50)
    k_stored, k_vec = dh.matrix_bytes(dk, dslot)
    k_bytes = k_stored + k_vec
    csr_bytes = 12 * dm.nnz + 4 * (dm.nrows + 1) + 8 * dm.ncols + 8 * dm.nrows
    peak, peak_src = peaks()
    achieved = k_bytes / (k_ms * 1e-3) / 1e9
    k_layout = dh.layout(dk, dslot) if plan is None else "partitioned"
    k_name = f"L{dk}.{dslot}"
    traffic = ncu_traffic(args.config, k_layout, k_name)
    lay_iter = layout_bytes_per_iter(dh, h) if plan is None else None
    line = {
        "metric": METRIC,
        "value": ms_iter,
        "unit": "ms/iter",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": tot_ms / max(args.steps, 1),
        "higher_is_better": False,
        "scaling": "strong" if (world > 1 and partitioned) else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generator + reference setup hierarchy)",
        "config": {
            "workload": WORKLOADS.get(args.config, args.config),
            "name": args.config,
            "parallelism": ("1 GPU" if world == 1 else
                            (f"row partition x{world} (NCCL halos, agglomeration below {args.agglom_rows} rows)"
                             if partitioned else f"replicas x{world}")),
            "step": "one PCG solve to rtol 1e-8 from x0=0, b resident in HBM",
            "l2": "inputs larger than L2 (hierarchy + vectors > 1 GB, per-iteration traffic >> 126 MB)",
            "levels": [int(l.a.nrows) for l in h.levels],
        },
        "iterations": iters[-1] if iters else None,
        "reference_iterations": ref_its,
        "final_true_relres": true_rel,
        "gflops": flops_iter / (ms_iter * 1e-3) / 1e9,
        "iteration_roofline": {
            "layout_bytes_per_iter": lay_iter,
            "layout_frac": (lay_iter / (ms_iter * 1e-3) / 1e9 / peak) if lay_iter else None,
            "model_bytes_per_iter": bytes_iter,
            "model_frac": bytes_iter / (ms_iter * 1e-3) / 1e9 / peak,
            "peak": peak,
            "note": ("layout_frac: bytes the chosen device layouts must stream per PCG iteration (same "
                     "application counts and vector terms as the SURVEY 8(d) model) / time / peak; model_frac: the "
                     "8(d) CSR model (12 B per stored entry), which the symmetric layout undercuts -- the BASELINE "
                     "north-star target (>= 0.60) is quoted on that model"),
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "kernel": (f"SpMV of {k_name} ({dm.nrows} rows, {dm.nnz} nnz; plain epilogue), device layout '{k_layout}': "
                       f"the largest share of an iteration ({dn} applications)"),
            "bytes_per_launch": k_bytes, "ms_per_launch": k_ms, "peak_source": peak_src,
            "iteration_share": [{"matrix": f"L{k}.{sl}", "ms_per_launch": t, "applications": n, "ms_per_iter": w}
                                for w, k, sl, t, n in shares[:8]],
            "note": ("achieved = bytes the layout must stream per launch (stored values + indices + x once + y "
                     "once, amg_matrix_bytes) / CUDA-event time of the launch; traffic = ncu dram bytes of one "
                     "launch from profiles/ncu_summary.json (null when not captured on this layout)"),
            "csr_model_bytes_per_launch": csr_bytes,
            "csr_model_gbs": csr_bytes / (k_ms * 1e-3) / 1e9,
        },
        "e2e": {"value": e2e_ms_iter, "unit": "ms/iter", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "mean": e2e_mean, "statistic": "median over the steps of (wall time of one pcg() call) / its iterations",
                "note": "whole job: every rank copies its slice of b in and of x out"},
        "gpu_launches": int(launches),
        "graph_mode": dh.stats()["graph_mode"],
        "clocks": clk.report(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dts = cpu_sample(h, b_host, args.cpu_iters, budget_s=30.0)
        line["cpu_baseline"] = {
            "value": float(np.mean(dts)), "unit": "ms/iter", "cores": 1, "kind": "port",
            "sample": f"{len(dts)} PCG iterations of the same workload (numpy oracle, bit-identical restatement "
                      "of the reference path), single-threaded",
            "host_cpu": _cpu_model(),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dh.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_amgb200(args)


if __name__ == "__main__":
    sys.exit(main())
