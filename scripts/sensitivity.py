"""Trajectory sensitivity of a TRON solve to last-bit perturbations (C -> C*(1+k*2^-52)):
GPU solves for k = 0..4 and, optionally, the reference CPU solver for k = 0, 1.
Shows whether CG-count / objective differences between two FP64 implementations
exceed what one implementation shows under a 1-ulp change of its input.
Usage: python scripts/sensitivity.py K1 [--reference]   (writes gpurun_out/sensitivity_<W>.json)"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, solve, synth
from paper_2008_03433_b200.tron import Problem

name = sys.argv[1] if len(sys.argv) > 1 else "K1"
with_ref = "--reference" in sys.argv
p0 = synth.make_shape(name)
loss = LossKind.Logistic if synth.SHAPES[name]["loss"] == "logistic" else LossKind.L2Svm
cfg = TrustRegionConfig(eps=0.01)
rows = []
base_w = None
for k in range(5):
    C = 1.0 * (1.0 + k * 2.0 ** -52)
    p = Problem(p0.X, p0.y, C)
    r = solve(p, loss, cfg, ExecutionPlan.gpu())
    if base_w is None:
        base_w = r.w
    rows.append({"impl": "b200", "k": k, "C": C, "objective": r.objective,
                 "cg_iters": [it.cg_iters for it in r.trace.iterations],
                 "rel_w_vs_k0": float(np.linalg.norm(r.w - base_w) / np.linalg.norm(base_w))})
    print(json.dumps(rows[-1]), flush=True)
if with_ref:
    from pyoracle import Reference
    ref = Reference()
    threads = min(len(os.sched_getaffinity(0)), 64)
    rw0 = None
    for k in (0, 1):
        C = 1.0 * (1.0 + k * 2.0 ** -52)
        t0 = time.time()
        w, t = ref.solve(Problem(p0.X, p0.y, C), 0 if loss == LossKind.Logistic else 1, cfg,
                         backend=Reference.PAR, workers=threads)
        if rw0 is None:
            rw0 = w
        rows.append({"impl": "reference", "k": k, "C": C, "objective": t["objective"],
                     "cg_iters": [it["cg_iters"] for it in t["iterations"]],
                     "rel_w_vs_k0": float(np.linalg.norm(w - rw0) / np.linalg.norm(rw0)),
                     "seconds": time.time() - t0})
        print(json.dumps(rows[-1]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(rows, open(os.path.join(ROOT, "gpurun_out", f"sensitivity_{name}.json"), "w"), indent=1)
