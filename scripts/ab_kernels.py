"""Kernel and solve times of one workload for A/B runs (variant libraries via
TRON_B200_LIB, switches via the environment): one JSON line.
  python scripts/ab_kernels.py W [tag]"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
W = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else ""
p = synth.make_shape(W, rows=int(os.environ["ROWS"]) if os.environ.get("ROWS") else None)
loss = LossKind.Logistic if synth.SHAPES[W]["loss"] == "logistic" else LossKind.L2Svm
with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
    cfg = TrustRegionConfig(eps=0.01)
    ev.solve(cfg)
    ts = []
    for _ in range(3):
        r = ev.solve(cfg)
        ts.append(r.device_ms)
    kt = ev.bench_kernels(reps=10, flush_l2=True)
nnz = p.X.stored()
hv_bytes = 24 * nnz + 32 * (p.X.rows + p.X.cols) if p.X.layout == "csr" else 8 * p.X.rows * p.X.cols + p.X.rows
print(json.dumps({"workload": W, "tag": tag, "lib": os.environ.get("TRON_B200_LIB", "default"),
                  "solve_ms": float(np.median(ts)), "hv_gbs": hv_bytes / (kt["hv_ms"] * 1e-3) / 1e9,
                  "objective": r.objective, "cg": [it.cg_iters for it in r.trace.iterations], **kt}), flush=True)
