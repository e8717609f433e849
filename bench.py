#!/usr/bin/env python
"""TRON time-to-eps on B200 (BASELINE.json metric) -- one JSON line.

A *step* is one complete TRON solve to eps (tron::solve, tron.cpp:127-217)
of the workload below, from w0 = 0, with the problem already resident in
HBM.  Default workload: BASELINE.json configs[1], the synthetic news20-shaped
sparse logistic regression (SYNTH-v1 N1: 19,996 x 1,355,191, 455 nnz/row,
C = 1, eps = 0.01, FP64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload N1|R1|P1|K1]
  python bench.py --impl reference ...   # the reference CPU solver (oracle/_ref)

For N > 1 (torchrun) the rows are sharded contiguously across ranks and the
per-call partial vectors are summed with NCCL (the north star's row-sharded
layout); time is the max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TRON train time to eps (s)"
UNIT = "s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, val in zip(names, r[3:7]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def workload_problem(name, rows=None):
    from paper_2008_03433_b200 import LossKind, synth
    s = synth.SHAPES[name]
    p = synth.make_shape(name, seed=1, rows=rows)
    loss = LossKind.Logistic if s["loss"] == "logistic" else LossKind.L2Svm
    return p, loss, s


def algorithmic_bytes(p, loss, active_frac=1.0):
    """SURVEY.md §8(d) algorithmic bytes per call (FP64 values, int32 indices)."""
    X = p.X
    l, n = X.rows, X.cols
    if X.layout == "csr":
        nnz = X.stored()
        return {"hv": 24 * nnz + 32 * (l + n), "fun": 12 * nnz + 8 * n + 40 * l,
                "grad": 12 * nnz + 24 * n + 8 * l, "transposed": 12 * nnz + 24 * n + 8 * l}
    hv = 8 * l * n + l  # masked traversal of column-major X + mask bytes
    return {"hv": hv, "fun": 8 * l * n + 17 * l, "grad": 8 * l * n + 17 * l, "transposed": hv}


def h2d_bytes(p):
    X = p.X
    b = X.values.nbytes + p.y.nbytes
    if X.layout == "csr":
        b += X.row_offsets.nbytes + X.col_indices.nbytes
    return int(b)


def pin_problem(p, torch):
    """Copy of a Problem whose arrays live in page-locked host memory."""
    from paper_2008_03433_b200.tron import FeatureMatrix, Problem

    def pinned(a):
        t = torch.empty(a.size, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        out = t.numpy()
        out[...] = a.reshape(-1)
        return out

    X = p.X
    if X.layout == "csr":
        Xp = FeatureMatrix("csr", X.rows, X.cols, pinned(X.values), pinned(X.row_offsets),
                           pinned(X.col_indices))
    else:
        Xp = FeatureMatrix("dense", X.rows, X.cols, pinned(X.values))
    return Problem(Xp, pinned(p.y), p.C)


def read_traffic(workload):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        return d.get(workload)
    except Exception:
        return None


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The reference's own CPU solver (proj/src, compiled in place into oracle/_ref)."""
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import REF_PATH, Reference, have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_PATH} not built"}))
        return 0
    if args.workload not in FULL_SOLVE_SAMPLE:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"a full reference solve of {args.workload} takes 10+ minutes on the host; the b200 "
                          "line's cpu_baseline carries the reference's per-call model instead"}))
        return 0
    from paper_2008_03433_b200 import TrustRegionConfig
    p, loss, s = workload_problem(args.workload)
    ref = Reference()
    threads = min(cpu_cores(), 64)  # the reference splits work into 64 tasks (parallel.hpp:24)
    cfg = TrustRegionConfig(eps=args.eps)
    oloss = 0 if loss.name == "Logistic" else 1
    for _ in range(args.warmup):
        ref.solve(p, oloss, cfg, backend=Reference.PAR, workers=threads)
    times = []
    t_obj = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        w, t = ref.solve(p, oloss, cfg, backend=Reference.PAR, workers=threads)
        times.append(time.perf_counter() - t0)
        t_obj = t
    v = float(np.mean(times))
    hv = sum(r["cg_iters"] for r in t_obj["iterations"])
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SYNTH-v1, seed 1)",
        "config": {"workload": args.workload, "shape": s["desc"], "C": 1.0, "eps": args.eps,
                   "backend": f"ExecutionPlan::parallel({threads})"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"full {args.workload} solve x{args.steps} (min {min(times):.3f} s)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "objective": t_obj["objective"], "hessian_products": hv,
        "outer_iterations": len(t_obj["iterations"]),
    }
    print(json.dumps(line))
    return 0


# Workloads whose full reference solve fits the bounded CPU sample (<= ~30 s
# on the box's 16 cores); the others are timed per call (see cpu_baseline).
FULL_SOLVE_SAMPLE = {"R1", "N1", "P1"}
PER_CALL_ROWS = {"Q1": 23_000_000}  # Q1: per-call costs on its first 2.3e7 rows, scaled by rows


def solve_call_counts(res):
    """fun / grad / Hv calls of a solve (tron.cpp:127-217 from the trace)."""
    it = res.trace.iterations if hasattr(res, "trace") else res["iterations"]
    acc = sum(1 for r in it if (r.accepted if hasattr(r, "accepted") else r["accepted"]))
    hv = sum((r.cg_iters if hasattr(r, "cg_iters") else r["cg_iters"]) for r in it)
    return 1 + len(it), 1 + acc, hv


def cpu_baseline(args, p_full, loss, cfg, res):
    """The reference CPU solver (oracle/_ref) on this host's cores, bounded.

    R1/N1/P1: full solves (min of up to 3 within ~20 s), with parity of the
    GPU result against it.  K1/Q1 (a full reference solve takes 10+ min):
    the reference evaluator's per-call cost (fun, grad, Hv at w = 0, the
    first outer iteration's state) times the solve's call counts; Q1's calls
    are timed on its first 2.3e7 rows and scaled by rows (dense: cost is
    linear in rows)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference, have_reference
    if not have_reference():
        return None
    ref = Reference()
    threads = min(cpu_cores(), 64)  # the reference splits work into 64 tasks (parallel.hpp:24)
    oloss = 0 if loss.name == "Logistic" else 1
    if args.workload in FULL_SOLVE_SAMPLE:
        ts = []
        t_begin = time.perf_counter()
        while len(ts) < 3 and (time.perf_counter() - t_begin) < 20.0:
            t0 = time.perf_counter()
            w_ref, t_ref = ref.solve(p_full, oloss, cfg, backend=Reference.PAR, workers=threads)
            ts.append(time.perf_counter() - t0)
        rel_f = abs(res.objective - t_ref["objective"]) / abs(t_ref["objective"])
        rel_w = float(np.linalg.norm(res.w - w_ref) / np.linalg.norm(w_ref))
        return {"value": float(min(ts)), "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"{len(ts)} full {args.workload} solves (min), ExecutionPlan::parallel({threads})",
                "parity": {"rel_objective": rel_f, "rel_w": rel_w,
                           "outer": [len(res.trace.iterations), len(t_ref["iterations"])],
                           "hv": [res.hessian_products, sum(r["cg_iters"] for r in t_ref["iterations"])]}}
    from paper_2008_03433_b200.tron import FeatureMatrix, Problem
    p_s, scale = p_full, 1.0
    rows = PER_CALL_ROWS.get(args.workload)
    if rows is not None and rows < p_full.X.rows:
        X = p_full.X
        p_s = Problem(FeatureMatrix("dense", rows, X.cols, X.values[: rows * X.cols]), p_full.y[:rows], p_full.C)
        scale = X.rows / rows
    t = ref.time_calls(p_s, oloss, threads, reps=1)
    n_fun, n_grad, n_hv = solve_call_counts(res)
    v = scale * (n_fun * t["fun_ms"] + n_grad * t["grad_ms"] + n_hv * t["hv_ms"]) / 1e3
    what = f"first {rows} rows, x{scale:.3f} by rows" if scale != 1.0 else "full problem"
    return {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": (f"per-call model: reference evaluator (ExecutionPlan::parallel({threads})) "
                       f"fun {t['fun_ms']:.1f} ms, grad {t['grad_ms']:.1f} ms, Hv {t['hv_ms']:.1f} ms "
                       f"at w=0 on the {what}, x the solve's calls ({n_fun} fun, {n_grad} grad, {n_hv} Hv)"),
            "per_call_ms": {k: float(x) for k, x in t.items()}}


# ---------------------------------------------------------------------------- B200 arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="N1", choices=["R1", "N1", "P1", "K1", "Q1"])
    ap.add_argument("--eps", type=float, default=0.01)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")

    if args.impl == "reference":
        rc = run_reference(args, rank, world)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return rc

    import ctypes

    from paper_2008_03433_b200 import ExecutionPlan, TrustRegionConfig, make_evaluator
    from paper_2008_03433_b200 import _lib
    from paper_2008_03433_b200.sharding import shard

    p_full, loss, s = workload_problem(args.workload)
    p, row_begin = shard(p_full, rank, world) if world > 1 else (p_full, 0)
    plan = ExecutionPlan.gpu(device=local_rank)
    if world > 1:
        uid = None
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            if _lib.lib.tron_gpu_nccl_unique_id(buf) != 0:
                raise RuntimeError(_lib.last_error())
            uid = buf.raw
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        plan.rank, plan.world, plan.nccl_unique_id = rank, world, obj[0]
        plan.row_begin, plan.global_rows = row_begin, p_full.X.rows
    cfg = TrustRegionConfig(eps=args.eps)

    import torch
    torch.cuda.set_device(local_rank)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    ev = make_evaluator(p, loss, plan)
    for _ in range(args.warmup):
        ev.solve(cfg)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    launches0 = ev.launch_count()
    step_ms, wall, res = [], [], None
    sampler = ClockSampler(local_rank)
    barrier()
    with sampler:
        for _ in range(args.steps):
            if flush is not None:  # inputs > L2 anyway for N1/K1/P1; flush for R1-sized cases
                flush.fill_(1)
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = ev.solve(cfg)
            wall.append(time.perf_counter() - t0)
            step_ms.append(res.device_ms)
    barrier()
    launches = ev.launch_count() - launches0
    t_step = float(np.mean(step_ms)) / 1e3  # CUDA-event time per solve on this rank
    if dist is not None:
        t = torch.tensor([t_step], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t[0])

    # ---- kernel-level roofline (dominant kernel: the Hessian-vector product)
    kt = ev.bench_kernels(reps=20, flush_l2=True)
    ab = algorithmic_bytes(p, loss)
    peak, peak_kind = load_peaks()
    hv_s = kt["hv_ms"] / 1e3
    achieved = ab["hv"] / hv_s / 1e9
    trans_gbs = ab["transposed"] / (kt["transposed_ms"] / 1e3) / 1e9

    # ---- e2e: the public API from pinned host buffers (create = H2D + on-device
    # CSC build, solve, w D2H), every step; the pinned copies are made untimed
    p_pin = pin_problem(p, torch) if args.workload != "Q1" else p  # Q1: 68.8 GB stays pageable
    e2e = []
    for k in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with make_evaluator(p_pin, loss, plan) as ev2:
            r2 = ev2.solve(cfg)
        e2e.append(time.perf_counter() - t0)
    del p_pin
    e2e_v = float(np.median(e2e))
    if dist is not None:
        t = torch.tensor([e2e_v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_v = float(t[0])

    if rank != 0:
        ev.close()
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- CPU baseline: the reference solver on this host, bounded sample
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(args, p_full, loss, cfg, res)

    nnz = p_full.X.stored()
    line = {
        "metric": METRIC, "value": t_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SYNTH-v1 generator, seed 1; SURVEY.md §8(d))",
        "config": {"workload": args.workload, "shape": s["desc"], "l": p_full.X.rows, "n": p_full.X.cols,
                   "nnz": nnz, "C": 1.0, "eps": args.eps, "loss": loss.name,
                   "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU",
                   "l2": "256 MiB flush before every step" if flush is not None else "no flush",
                   "timing": "CUDA events on the solver stream around each solve, mean over steps"},
        "objective": res.objective, "converged": res.converged,
        "outer_iterations": len(res.trace.iterations), "hessian_products": res.hessian_products,
        "hv_per_s": res.hessian_products / t_step if t_step > 0 else None,
        "wall_ms_per_step": float(np.mean(wall)) * 1e3,
        "roofline": {"bound": "hbm",
                     "kernel": ("Hessian-vector product (CSR D*Xv + CSC segmented X^T u)" if p.X.layout == "csr"
                                else "Hessian-vector product (dense tall-skinny TMA pass, one read of X)"),
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": f"{peak_kind} (copy read+write GB/s; frac is 'of {peak_kind}')",
                     "traffic": read_traffic(args.workload),
                     "algorithmic_bytes_per_launch": ab["hv"], "avg_launch_ms": kt["hv_ms"],
                     "launch_timing": "CUDA events around each Hv launch on the solver stream, 256 MiB "
                                      "L2 flush before each, mean of 20, same process after the timed solves",
                     "hv_share_of_step": res.hessian_products * kt["hv_ms"] / (t_step * 1e3) if t_step > 0 else None,
                     "transposed_only_gbs": trans_gbs, "kernel_ms": kt},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes(p),
                "d2h_bytes_per_step": int(8 * p.X.cols + 64),
                "what": ("make_evaluator from " + ("pageable (staged)" if args.workload == "Q1" else "pinned")
                         + " host arrays (H2D + device CSC build / transpose) + solve + w to host + destroy, via the C ABI")},
        "gpu_launches": int(launches),
        "clocks": sampler.summary(),
        "device_memory_bytes": ev.memory_bytes(),
    }
    print(json.dumps(line))
    ev.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
