#!/usr/bin/env python
"""TRON time-to-eps on B200 (BASELINE.json metric) -- one JSON line.

A *step* is one complete TRON solve to eps (tron::solve, tron.cpp:127-217)
of the workload below, from w0 = 0, with the problem already resident in
HBM; ``value`` is the host wall time of that solve call (the boundary of
cli.cpp:215-218: the call returns with w on the host).  Default workload:
BASELINE.json configs[2], the largest single-GPU configuration -- the
synthetic proteomics-shaped L2-SVM (SYNTH-v1 P1: 2.3e7 x 40 dense, C = 1,
eps = 0.01, FP64).  R1/N1 (sparse LR) and K1/Q1 (the 1/2/4/8-GPU configs)
are selectable with --workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload P1|R1|N1|K1|Q1]
  python bench.py --impl reference ...   # the reference CPU solver (oracle/_ref only)

For N > 1 the rows are sharded contiguously across ranks and the per-call
partial vectors are summed with NCCL (the north star's row-sharded layout);
time is the max over ranks.  Without torchrun, ``--gpus N`` (N > 1) re-launches
itself under torch.distributed.run.

The reference arm never maps the product library: its inputs come from the
SYNTH-v1 generator inside oracle/_ref (the reference's own testgen::Rng).
"""
import argparse
import gc
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TRON train time to eps (s)"
FP64_TENSOR_TFLOPS = 45.0  # B200 nominal (no measured FP64 figure in MEASURED_PEAKS.json)
UNIT = "s"
SEED = 1
TEST_SEED = 2  # held-out rows for the prediction parity check

# SYNTH-v1 shapes (BASELINE.json configs).  Kept here so the
# reference arm does not import the product package (tests check it equals
# paper_2008_03433_b200.synth.SHAPES).
SHAPES = {
    "R1": dict(kind="sparse", l=20242, n=47236, k=74, loss="logistic",
               desc="rcv1-shaped sparse LR 20,242x47,236, 74 nnz/row"),
    "N1": dict(kind="sparse", l=19996, n=1355191, k=455, loss="logistic",
               desc="news20-shaped sparse LR 19,996x1,355,191, 455 nnz/row"),
    "P1": dict(kind="dense", l=23_000_000, n=40, loss="l2svm",
               desc="proteomics-shaped dense L2-SVM 2.3e7x40"),
    "K1": dict(kind="sparse", l=8_400_000, n=20_000_000, k=36, loss="logistic",
               desc="kdd2010-shaped sparse LR 8.4e6x2.0e7, 36 nnz/row"),
    "Q1": dict(kind="dense", l=215_000_000, n=40, loss="l2svm",
               desc="quarter-billion dense L2-SVM 2.15e8x40"),
}
# Full reference solves that fit the bounded CPU sample (<= ~30 s on 16 cores).
FULL_SOLVE_SAMPLE = {"R1", "N1", "P1"}
PARITY_FILES = {"K1": "profiles/parity_K1.json", "Q1": "profiles/parity_Q1.json"}


def workload_config(name, eps, rows=None):
    """The config dict both arms print (identical by construction)."""
    s = SHAPES[name]
    l = rows if rows is not None else s["l"]
    nnz = l * (s["k"] if s["kind"] == "sparse" else s["n"])
    return {"workload": name, "shape": s["desc"] + (f", first {l} rows" if rows is not None else ""),
            "l": l, "n": s["n"], "nnz": nnz, "C": 1.0,
            "eps": eps, "loss": "Logistic" if s["loss"] == "logistic" else "L2Svm", "w0": "zeros",
            "generator": f"SYNTH-v1 seed {SEED}",
            "l2": ("inputs larger than L2 (126 MB) and a 256 MiB read-based L2 eviction before every "
                   "step" if (nnz * 12 > 126e6) else "256 MiB read-based L2 eviction before every step")}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_description():
    model, mem_gb = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_gb = round(int(line.split()[1]) / 2**20, 1)
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "usable_cores": cpu_cores(), "mem_gb": mem_gb}


def _nvml_sampler_proc(device_uuid, device_index, conn, stop, go, ready):
    """Child process: SM clocks + throttle-reason bits every 20 ms while `go` is
    set (the timed region), until `stop`; then the samples through `conn`.  A separate process shares no GIL
    with the timed loop (an in-process sampler thread delayed the return of
    1-2 ms solves by holding the GIL across NVML calls)."""
    rows = []
    try:
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByUUID(device_uuid) if device_uuid else nv.nvmlDeviceGetHandleByIndex(device_index)
        except Exception:
            h = nv.nvmlDeviceGetHandleByIndex(device_index)
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        # every query once before the timed region: a first call can hold the
        # driver for tens of ms (it stalled the second timed solve)
        nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get(h)
        ready.set()
        while not stop.is_set():
            if go.is_set():
                try:
                    rows.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                 float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)), int(get(h))))
                except Exception:
                    pass
            stop.wait(0.02)
    except Exception:
        pass
    ready.set()
    conn.send(rows)
    conn.close()


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, by an NVML
    child process (nvidia-smi only if NVML is unavailable)."""

    # nvmlClocksEventReasons bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, set of reasons)
        self.source = "nvml"
        try:
            import pynvml  # noqa: F401
        except Exception:
            self.source = "nvidia-smi"

    def _smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        r = [x.strip() for x in out.split(",")]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return float(r[0]), float(r[1]), {n for n, v in zip(names, r[3:7]) if v.lower() == "active"}

    def __enter__(self):
        if os.environ.get("TRON_BENCH_NO_SAMPLER") == "1":  # (diagnostics: one nvidia-smi read at the end)
            self.source = "nvidia-smi"
            return self
        if self.source == "nvml":
            import multiprocessing as mp
            uuid = None
            try:
                import torch
                u = str(torch.cuda.get_device_properties(self.device).uuid)
                uuid = u if u.startswith("GPU-") else "GPU-" + u
            except Exception:
                pass
            ctx = mp.get_context("spawn")
            self._rx, tx = ctx.Pipe(duplex=False)
            self._stop, self._go, ready = ctx.Event(), ctx.Event(), ctx.Event()
            self._proc = ctx.Process(target=_nvml_sampler_proc,
                                     args=(uuid, self.device, tx, self._stop, self._go, ready), daemon=True)
            self._proc.start()
            ready.wait(60)  # NVML initialised and every query made once before the timed region
            time.sleep(0.1)
            self._go.set()
        return self

    def __exit__(self, *exc):
        if self.source == "nvml":
            self._go.clear()
            self._stop.set()
            try:
                if self._rx.poll(30):
                    raw = self._rx.recv()
                    self.rows = [(a, b, {nm for bit, nm in self.REASONS.items() if r & bit}) for a, b, r in raw]
            except Exception:
                pass
            self._proc.join(timeout=10)
        if not self.rows:
            try:
                self.rows = [self._smi()]
                self.source = "nvidia-smi (after the timed region)"
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = set().union(*(r[2] for r in self.rows))
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": sorted(reasons),
                "samples": len(self.rows), "source": self.source}


# ---------------------------------------------------------------------------- oracle-side data

class _Matrix:  # the attributes pyoracle reads (FeatureMatrix-like)
    def __init__(self, layout, rows, cols, values, row_offsets=None, col_indices=None):
        self.layout, self.rows, self.cols = layout, rows, cols
        self.values, self.row_offsets, self.col_indices = values, row_offsets, col_indices

    def stored(self):
        return self.values.size


class _Problem:
    def __init__(self, X, y, C=1.0):
        self.X, self.y, self.C = X, y, C


def oracle_problem(ref, name, seed=SEED, rows=None):
    """SYNTH-v1 problem generated inside oracle/_ref (no product library)."""
    s = SHAPES[name]
    l = rows if rows is not None else s["l"]
    if s["kind"] == "sparse":
        ro, ci, vals, y = ref.synth_sparse(seed, l, s["n"], s["k"])
        return _Problem(_Matrix("csr", l, s["n"], vals, ro, ci), y)
    vals, y = ref.synth_dense(seed, l, s["n"])
    return _Problem(_Matrix("dense", l, s["n"], vals), y)


def ref_loss(name):
    return 0 if SHAPES[name]["loss"] == "logistic" else 1


def ref_cfg(eps):
    from pyoracle import make_config
    return make_config(None, eps=eps)


def counts_of(trace_iters):
    return {"outer": len(trace_iters), "accepted": sum(1 for r in trace_iters if r["accepted"]),
            "cg_iters": [int(r["cg_iters"]) for r in trace_iters]}


def modelled_reference_solve(ref, p, name, threads):
    """K1/Q1: a full reference solve takes 9-10 minutes (K1) or needs ~140 GB
    of host RAM (Q1), so a step is the reference evaluator's measured per-call
    cost (fun, grad, Hv at w = 0; Q1 on its first 2.3e7 rows, scaled by rows)
    times the call counts of the measured full reference solve recorded in
    profiles/parity_<W>.json."""
    rec = json.load(open(os.path.join(ROOT, PARITY_FILES[name])))
    rc = rec["reference"]  # scripts/parity_run.py format
    n_fun, n_grad, n_hv = 1 + rc["outer"], 1 + rc["accepted"], sum(rc["cg_iters"])
    p_s, scale = p, 1.0
    if name == "Q1":
        rows = 23_000_000
        X = p.X
        p_s = _Problem(_Matrix("dense", rows, X.cols, X.values[: rows * X.cols]), p.y[:rows])
        scale = X.rows / rows
    t = ref.time_calls(p_s, ref_loss(name), threads, reps=1)
    v = scale * (n_fun * t["fun_ms"] + n_grad * t["grad_ms"] + n_hv * t["hv_ms"]) / 1e3
    return v, (f"per-call model: reference evaluator ExecutionPlan::parallel({threads}) fun "
               f"{t['fun_ms']:.1f} ms, grad {t['grad_ms']:.1f} ms, Hv {t['hv_ms']:.1f} ms at w=0"
               + (f" on the first {23_000_000} rows x{scale:.3f}" if scale != 1.0 else "")
               + f", x the measured reference solve's calls ({n_fun} fun, {n_grad} grad, {n_hv} Hv; "
               f"{PARITY_FILES[name]})")


# ---------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The reference's own CPU solver (proj/src, compiled in place into
    oracle/_ref) through its public tron::solve, ExecutionPlan::parallel(T)."""
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import REF_PATH, Reference, have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_PATH} not built"}))
        return 0
    ref = Reference()
    threads = min(cpu_cores(), 64)  # the reference splits work into 64 tasks (parallel.hpp:24)
    p = oracle_problem(ref, args.workload, rows=args.rows)
    cfg = ref_cfg(args.eps)
    loss = ref_loss(args.workload)
    extra = {}
    if args.workload in FULL_SOLVE_SAMPLE or args.rows is not None:
        for _ in range(args.warmup):
            ref.solve(p, loss, cfg, backend=Reference.PAR, workers=threads)
        times, t_obj = [], None
        for _ in range(args.steps):
            t0 = time.perf_counter()
            w, t_obj = ref.solve(p, loss, cfg, backend=Reference.PAR, workers=threads)
            times.append(time.perf_counter() - t0)
        v = float(np.mean(times))
        sample = f"full {args.workload} solve x{args.steps} (mean; min {min(times):.4f} s)"
        extra = {"objective": t_obj["objective"], "hessian_products": sum(counts_of(t_obj["iterations"])["cg_iters"]),
                 "outer_iterations": len(t_obj["iterations"]), "wall_min_s": min(times)}
    else:
        vs = []
        for _ in range(args.warmup + args.steps):
            v, sample = modelled_reference_solve(ref, p, args.workload, threads)
            vs.append(v)
        v = float(np.mean(vs[args.warmup:]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (SYNTH-v1 seed {SEED}, generated inside oracle/_ref)",
        "config": workload_config(args.workload, args.eps, args.rows),
        "backend": f"ExecutionPlan::parallel({threads}) on the host CPU",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                         "host": host_description()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------- B200 arm helpers

def product_problem(name, seed=SEED, rows=None):
    from paper_2008_03433_b200 import LossKind, synth
    s = SHAPES[name]
    p = synth.make_shape(name, seed=seed, rows=rows)
    return p, (LossKind.Logistic if s["loss"] == "logistic" else LossKind.L2Svm)


def algorithmic_bytes(p):
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
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(workload)
    except Exception:
        return None


def cpu_baseline(args, p_full, res, ev, loss, cfg, plan, act_gpu=None):
    """The reference CPU solver (oracle/_ref) on this host's cores, bounded,
    plus the parity of the GPU result against it (north-star gate)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference, have_reference
    if not have_reference():
        return None
    ref = Reference()
    threads = min(cpu_cores(), 64)  # the reference splits work into 64 tasks (parallel.hpp:24)
    oloss = ref_loss(args.workload)
    rcfg = ref_cfg(args.eps)
    out = {"unit": UNIT, "cores": threads, "kind": "reference", "host": host_description()}
    if args.workload not in FULL_SOLVE_SAMPLE and args.rows is None:
        v, sample = modelled_reference_solve(ref, p_full, args.workload, threads)
        out.update(value=v, sample=sample)
        try:
            rec = json.load(open(os.path.join(ROOT, PARITY_FILES[args.workload])))
            out["parity"] = rec["parity"]
            out["parity"]["source"] = PARITY_FILES[args.workload] + " (full-size run, same generator)"
            # the measured full reference solve behind the model (same SYNTH-v1 input)
            secs = rec.get("reference_solve_s") or rec.get("reference", {}).get("seconds")
            if secs:
                out["full_solve_measured_s"] = secs
                out["full_solve_measured_where"] = (f"{PARITY_FILES[args.workload]}: ExecutionPlan::parallel("
                                                    f"{rec.get('threads', '?')}) "
                                                    + ("on this pool's GPU box" if args.workload == "Q1"
                                                       else "in the build container (8 cores)"))
            if "tight" in rec:
                out["parity"]["tight_eps"] = {k: rec["tight"][k] for k in ("eps", "rel_objective", "rel_w")
                                              if k in rec["tight"]}
        except Exception:
            pass
        return out
    ts = []
    t_begin = time.perf_counter()
    while len(ts) < 3 and (time.perf_counter() - t_begin) < 25.0:
        t0 = time.perf_counter()
        w_ref, t_ref = ref.solve(p_full, oloss, rcfg, backend=Reference.PAR, workers=threads)
        ts.append(time.perf_counter() - t0)
    out.update(value=float(min(ts)),
               sample=f"{len(ts)} full {args.workload} solves (min), ExecutionPlan::parallel({threads})")
    # the 1-core leg: ExecutionPlan::sequential() -- a full solve when the
    # parallel one is short, else the per-call model on a row sample
    if ts[0] < 2.0:
        t0 = time.perf_counter()
        ref.solve(p_full, oloss, rcfg, backend=Reference.SEQ, workers=1)
        out["sequential"] = {"value": time.perf_counter() - t0, "cores": 1,
                             "sample": f"1 full {args.workload} solve, ExecutionPlan::sequential()"}
    elif p_full.X.layout == "dense":
        from paper_2008_03433_b200.tron import FeatureMatrix, Problem
        X = p_full.X
        rows = X.rows // 10
        p_s = Problem(FeatureMatrix("dense", rows, X.cols, X.values[: rows * X.cols]), p_full.y[:rows], 1.0)
        t = ref.time_calls(p_s, oloss, 1, reps=1, backend=Reference.SEQ)
        c = counts_of(t_ref["iterations"])
        n_fun, n_grad, n_hv = 1 + c["outer"], 1 + c["accepted"], sum(c["cg_iters"])
        out["sequential"] = {"value": 10 * (n_fun * t["fun_ms"] + n_grad * t["grad_ms"] + n_hv * t["hv_ms"]) / 1e3,
                             "cores": 1,
                             "sample": (f"per-call model: ExecutionPlan::sequential() fun {t['fun_ms']:.0f} ms, "
                                        f"grad {t['grad_ms']:.0f} ms, Hv {t['hv_ms']:.0f} ms at w=0 on the first "
                                        f"{rows} rows x10, x the reference solve's calls")}
    # ---- parity (BASELINE.json north star): objective and w within 1e-6,
    # counts within +-1, SVM active sets and test predictions identical
    it_gpu = [{"accepted": r.accepted, "cg_iters": r.cg_iters} for r in res.trace.iterations]
    cg, cr = counts_of(it_gpu), counts_of(t_ref["iterations"])
    rel_f = abs(res.objective - t_ref["objective"]) / abs(t_ref["objective"])
    rel_w = float(np.linalg.norm(res.w - w_ref) / np.linalg.norm(w_ref))
    par = {"rel_objective": rel_f, "rel_w": rel_w, "outer": [cg["outer"], cr["outer"]],
           "accepted": [cg["accepted"], cr["accepted"]], "cg_iters": [cg["cg_iters"], cr["cg_iters"]],
           "hv": [sum(cg["cg_iters"]), sum(cr["cg_iters"])]}
    par["gate_pass"] = bool(rel_f <= 1e-6 and rel_w <= 1e-6 and abs(cg["outer"] - cr["outer"]) <= 1
                            and all(abs(a - b) <= 1 for a, b in zip(cg["cg_iters"], cr["cg_iters"]))
                            and len(cg["cg_iters"]) == len(cr["cg_iters"]))
    if oloss == 1:  # SVM active set I = {i : 1 - y_i z_i > 0} at each solver's final w
        sharded = act_gpu is not None  # the ranks' local sets, concatenated in rank order
        if not sharded:
            act_gpu = ev.committed_state().active
        act_ref = ref.svm(p_full, w_ref, np.zeros(p_full.X.cols))["active"]
        par["active_set_identical"] = bool(np.array_equal(act_gpu, act_ref))
        par["active_set_sizes"] = [int(act_gpu.size), int(act_ref.size)]
        par["active_set_symmetric_difference"] = int(np.setxor1d(act_gpu, act_ref).size)
        if not sharded:
            ev.eval_candidate(w_ref)  # the GPU margin pass at the reference's w: bit-exact rows
            par["active_set_identical_at_reference_w"] = bool(
                np.array_equal(ev.candidate_state().active, act_ref))
    # predictions (model.cpp:88-117) on held-out SYNTH-v1 rows (seed 2)
    from paper_2008_03433_b200 import ExecutionPlan, make_evaluator
    test_rows = min(p_full.X.rows, 2_000_000)
    p_test, _ = product_problem(args.workload, seed=TEST_SEED, rows=test_rows)
    with make_evaluator(p_test, loss, ExecutionPlan.gpu(device=plan.device)) as evt:
        lab_gpu, correct_gpu = evt.predict(res.w)
        lab_gpu_at_ref, _ = evt.predict(w_ref)
    Xt = p_test.X
    Xt.y = p_test.y
    lab_ref, correct_ref = ref.predict(Xt, w_ref)
    par["predictions_identical"] = bool(np.array_equal(lab_gpu, lab_ref))
    par["predictions_differing"] = int(np.sum(lab_gpu != lab_ref))
    par["predictions_identical_at_reference_w"] = bool(np.array_equal(lab_gpu_at_ref, lab_ref))
    par["test_rows"] = test_rows
    par["test_accuracy"] = [correct_gpu / test_rows, correct_ref / test_rows]
    if oloss == 1 and p_full.X.layout == "dense" and p_full.X.cols <= 48:
        # the bit-for-bit mode: every reduction in the reference's order (refexact.cu)
        with make_evaluator(p_full, loss, ExecutionPlan.gpu(device=plan.device, reference_order=True)) as evr:
            evr.solve(cfg)  # warm (graph instantiation)
            t0 = time.perf_counter()
            r3 = evr.solve(cfg)
            t_ro = time.perf_counter() - t0
            act_ro = evr.committed_state().active
        lab_ro, _ = ref.predict(Xt, r3.w)
        c3 = counts_of([{"accepted": r.accepted, "cg_iters": r.cg_iters} for r in r3.trace.iterations])
        par["reference_order"] = {
            "what": "same solve with ExecutionPlan.gpu(reference_order=True): the reference's 64-block "
                    "chains + pairwise tree and serial n-dots (refexact.cu)",
            "solve_s": t_ro,
            "w_bitwise_identical": bool(np.array_equal(r3.w.view(np.uint64), w_ref.view(np.uint64))),
            "objective_bitwise_identical": bool(r3.objective == t_ref["objective"]),
            "counts_identical": c3 == cr,
            "active_set_identical": bool(np.array_equal(act_ro, act_ref)),
            "predictions_identical": bool(np.array_equal(lab_ro, lab_ref)),
        }
    out["parity"] = par
    return out


def spawn_ranks(args):
    """--gpus N without torchrun: re-launch under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------- B200 arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="P1", choices=list(SHAPES))
    ap.add_argument("--eps", type=float, default=0.01)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--rows", type=int, default=None,
                    help="first ROWS rows of the workload only (tests; the config says so)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="N > 1 data plane: NCCL (one GPU per rank) or the host allreduce over the gloo "
                         "group (ranks may share a GPU: a functional check of the N > 1 flow)")
    args = ap.parse_args()
    if os.environ.get("TRON_BENCH_WATCHDOG") and "WORLD_SIZE" in os.environ:
        # debugging: every thread's stack after N s into gpurun_out/hang_rank<R>.txt, then exit
        import faulthandler
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        _wd = open(os.path.join(ROOT, "gpurun_out", f"hang_rank{os.environ.get('RANK', '0')}.txt"), "w")
        faulthandler.dump_traceback_later(int(os.environ["TRON_BENCH_WATCHDOG"]), exit=True, file=_wd)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import ctypes

    import torch
    import torch.distributed as dist_mod

    from paper_2008_03433_b200 import ExecutionPlan, TrustRegionConfig, make_evaluator
    from paper_2008_03433_b200 import _lib
    from paper_2008_03433_b200.sharding import shard

    dist = None
    if world > 1:
        dist = dist_mod
        dist.init_process_group("gloo")

    p_full, loss = product_problem(args.workload, rows=args.rows)
    p, row_begin = shard(p_full, rank, world) if world > 1 else (p_full, 0)

    device = local_rank % max(torch.cuda.device_count(), 1)

    def make_plan():
        """The rank's plan; N > 1: a fresh NCCL unique id (rank 0's, broadcast)
        for every context -- an id serves one communicator -- or the host
        data plane over the gloo group."""
        pl = ExecutionPlan.gpu(device=device)
        if world > 1 and args.comm == "host":
            pl.rank, pl.world = rank, world
            pl.row_begin, pl.global_rows = row_begin, p_full.X.rows
            pl.host_allreduce = lambda buf: dist.all_reduce(torch.from_numpy(buf))
            return pl
        if world > 1:
            uid = None
            if rank == 0:
                buf = ctypes.create_string_buffer(128)
                if _lib.lib.tron_gpu_nccl_unique_id(buf) != 0:
                    raise RuntimeError(_lib.last_error())
                uid = buf.raw
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            pl.rank, pl.world, pl.nccl_unique_id = rank, world, obj[0]
            pl.row_begin, pl.global_rows = row_begin, p_full.X.rows
        return pl

    plan = make_plan()
    cfg = TrustRegionConfig(eps=args.eps)

    torch.cuda.set_device(device)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def evict_l2():  # read-based: leaves nothing dirty to write back inside the step
        if flush is not None:
            flush.view(torch.int64).sum()
        torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    ev = make_evaluator(p, loss, plan)
    for _ in range(args.warmup):
        ev.solve(cfg)

    launches0 = ev.launch_count()
    wall, dev_ms, res = [], [], None
    sampler = ClockSampler(device)
    barrier()
    gc.disable()  # (as timeit does: a collector pause is host noise, not the solve)
    with sampler:
        for _ in range(args.steps):
            evict_l2()
            t0 = time.perf_counter()
            res = ev.solve(cfg)  # returns with w in host memory
            wall.append(time.perf_counter() - t0)
            dev_ms.append(res.device_ms)
    gc.enable()
    barrier()
    launches = ev.launch_count() - launches0
    t_step = max_over_ranks(float(np.mean(wall)))
    t_dev = max_over_ranks(float(np.mean(dev_ms)) / 1e3)

    # ---- kernel-level roofline (dominant kernel: the Hessian-vector product)
    kt = ev.bench_kernels(reps=20, flush_l2=True)
    ab = algorithmic_bytes(p)
    peak, peak_kind = load_peaks()
    mode = ev.mode()
    trans_gbs = ab["transposed"] / (kt["transposed_ms"] / 1e3) / 1e9
    n_evals = res.trace.objective_evaluations
    if p.X.layout == "dense" and mode["gram"]:
        # Hessian as an n x n matrix per commit (gram.cu): the CG's Hv no longer
        # reads X; the passes over X are the fused margin pass (one per
        # evaluation; gram_delta: it also adds the rows that changed side to the
        # committed G) and the Gram pass (gram_delta: at w0 only; else once per
        # committed iterate that runs a CG).  The roofline object describes the
        # one with the larger share of the solve.
        l, n = p.X.rows, p.X.cols
        fwd_bytes = 8 * l * n + (18 if mode.get("gram_delta") else 17) * l
        gram_bytes = fwd_bytes if mode.get("gram_delta") else 8 * l * n + l
        gram_flops = l * n * (n + 1)  # the upper triangle of sum_i c_i x_i x_i^T, 2 flops per product
        n_gram = 1 if mode.get("gram_delta") else max(1, res.trace.accepted_steps)
        delta = bool(mode.get("gram_delta"))
        n_fwd = n_evals - 1 if delta else n_evals  # (delta: the first margin pass is the Gram pass)
        if n_gram * kt["grad_ms"] >= n_fwd * kt["forward_ms"]:
            # bound by the FP64 tensor pipe (ncu: math-pipe throttle), HBM a close second
            kern = ("first margin pass, forming the whole G = sum_i c_i x_i x_i^T on the FP64 tensor cores "
                    "(dense_pass PM_FWDD, empty reference)" if delta else
                    "Gram pass G = sum_i c_i x_i x_i^T (gram.cu, DMMA; once per commit)")
            kbytes, kms = gram_bytes, kt["grad_ms"]
            bound, unit = "tensor", "TFLOP/s"
            achieved = gram_flops / (kms / 1e3) / 1e12
            peak, peak_kind = FP64_TENSOR_TFLOPS, ("fallback: B200 FP64 tensor 45 TFLOPS "
                                                   "(/opt/skills/guides/blackwell_cuda_programming.md:52)")
        else:
            kern = ("fused margin pass (dense_pass FWDD: margins, mask, f, gradient partials, and the rows "
                    "that changed side added to the committed G)" if delta else
                    "fused margin pass (dense_pass FWD: margins, mask, f, gradient partials)")
            kbytes, kms = fwd_bytes, kt["forward_ms"]
            bound, unit = "hbm", "GB/s"
            achieved = kbytes / (kms / 1e3) / 1e9
        share = (n_gram if bound == "tensor" else n_fwd) * kms / (t_step * 1e3) if t_step > 0 else None
        gram_extra = {"gram_delta": bool(mode.get("gram_delta")), "gram_passes_per_solve": n_gram,
                      "gram_pass_ms": kt["grad_ms"], "gram_pass_hbm_gbs": gram_bytes / (kt["grad_ms"] / 1e3) / 1e9,
                      "gram_pass_fp64_tflops": gram_flops / (kt["grad_ms"] / 1e3) / 1e12,
                      "margin_pass_what": ("a candidate pass at the iterate before the last commit against the committed G: "
                                           "it adds the rows of the last commit's change (P1: 1.8% of rows; the solve's "
                                           "earlier passes change 6-11%)" if delta else "margin pass at the committed w"),
                      "margin_pass_ms": kt["forward_ms"], "margin_pass_gbs": fwd_bytes / (kt["forward_ms"] / 1e3) / 1e9,
                      "hv_from_gram_us": kt["hv_ms"] * 1e3,
                      "tall_skinny_hv_pass_ms": kt["transposed_ms"], "tall_skinny_hv_gbs": trans_gbs}
    else:
        kern = ("Hessian-vector product (CSR D*Xv + CSC segmented X^T u)" if p.X.layout == "csr"
                else "Hessian-vector product (dense tall-skinny TMA pass, one read of X)")
        kbytes, kms = ab["hv"], kt["hv_ms"]
        bound, unit = "hbm", "GB/s"
        achieved = kbytes / (kms / 1e3) / 1e9
        share = res.hessian_products * kms / (t_step * 1e3) if t_step > 0 else None
        gram_extra = {}

    # ---- e2e through the public API, every step: make_evaluator from the
    # caller's PAGEABLE numpy arrays (H2D + on-device CSC build / transpose),
    # solve, w to host, destroy.  The pinned-input variant is an extra key.
    def e2e_time(prob, reps):
        ts = []
        for _ in range(reps):
            pl = make_plan()  # (N > 1: its id broadcast happens before the timer)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with make_evaluator(prob, loss, pl) as ev2:
                ev2.solve(cfg)
            ts.append(time.perf_counter() - t0)
        return max_over_ranks(float(np.median(ts)))

    reps = max(2, min(args.steps, 5))
    e2e_v = e2e_time(p, reps)
    e2e_pin = None
    if args.workload != "Q1":  # Q1's 68.8 GB is not duplicated into pinned memory
        p_pin = pin_problem(p, torch)
        e2e_pin = e2e_time(p_pin, reps)
        del p_pin

    replicas_identical = None
    if world > 1:  # the replicated w must be bit-identical on every rank
        import hashlib
        digests = [None] * world
        dist.all_gather_object(digests, hashlib.sha1(np.ascontiguousarray(res.w).tobytes()).hexdigest())
        replicas_identical = len(set(digests)) == 1
    cpu = None
    act_all = None
    if world > 1 and not args.no_cpu_baseline and SHAPES[args.workload]["loss"] == "l2svm":
        parts = [None] * world  # every rank's local active set (global row ids)
        dist.all_gather_object(parts, ev.committed_state().active)
        act_all = np.concatenate(parts)
    if rank == 0 and not args.no_cpu_baseline:
        # (N > 1: rank 0 alone, the other ranks wait at the closing barrier)
        cpu = cpu_baseline(args, p_full, res, ev, loss, cfg, plan, act_gpu=act_all)

    # (every collective happens before the ranks part: the other ranks wait at
    # the closing barrier while rank 0 assembles the line)
    wall_min = max_over_ranks(float(np.min(wall)))
    if rank != 0:
        ev.close()
        barrier()
        dist.destroy_process_group()
        return 0

    line = {
        "metric": METRIC, "value": t_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (SYNTH-v1 generator, seed {SEED}; SURVEY.md §8(d))",
        "config": workload_config(args.workload, args.eps, args.rows),
        "parallelism": (f"row-sharded x{world} ({'NCCL' if args.comm == 'nccl' else 'host/gloo'} allreduce of "
                        "partials)") if world > 1 else "1 GPU",
        "timing": ("value: host wall time of each solve call (returns with w on the host), mean over "
                   "steps, max over ranks; device_s: CUDA-event time of the same solves"),
        "device_s": t_dev, "wall_s_min": wall_min, "wall_ms_steps": [round(x * 1e3, 3) for x in wall],
        "objective": res.objective, "converged": res.converged,
        "outer_iterations": len(res.trace.iterations), "hessian_products": res.hessian_products,
        "hv_per_s": res.hessian_products / t_step if t_step > 0 else None,
        "roofline": {"bound": bound, "kernel": kern,
                     "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                     "peak_source": (peak_kind if bound == "tensor" else
                                     f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs: copy read+write GB/s)"),
                     "traffic": read_traffic(args.workload + ("" if not gram_extra else
                                                             "-gram-delta" if gram_extra.get("gram_delta") and bound == "hbm"
                                                             else "-gram")),
                     "algorithmic_bytes_per_launch": kbytes, "avg_launch_ms": kms,
                     "launch_timing": "CUDA events around each launch on the solver stream, 256 MiB "
                                      "read-based L2 eviction before each, mean of 20, after the timed solves",
                     "share_of_step": share,
                     "transposed_only_gbs": trans_gbs, "kernel_ms": kt, **gram_extra},
        "mode": mode,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes(p),
                "d2h_bytes_per_step": int(8 * p.X.cols + 64),
                "what": ("make_evaluator from the caller's pageable numpy arrays (H2D + on-device CSC build / "
                         "transpose) + solve + w to host + destroy, through the C ABI; median of "
                         f"{reps}"),
                "pinned_inputs_value": e2e_pin},
        "replica_w_bitwise_identical": replicas_identical,
        "gpu_launches": int(launches),
        "clocks": sampler.summary(),
        "device_memory_bytes": ev.memory_bytes(),
    }
    print(json.dumps(line))
    ev.close()
    if dist is not None:
        barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
