"""Full-size parity of the B200 solve against the reference CPU solver (oracle/_ref)
on the same SYNTH-v1 input: objective, w, outer / accepted / per-iteration CG counts.
Usage: python scripts/parity_full.py K1 [threads]   (writes gpurun_out/parity_<W>.json)"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, solve, synth
from pyoracle import Reference

name = sys.argv[1] if len(sys.argv) > 1 else "K1"
threads = int(sys.argv[2]) if len(sys.argv) > 2 else min(len(os.sched_getaffinity(0)), 64)
t0 = time.time()
p = synth.make_shape(name)
gen_s = time.time() - t0
loss = LossKind.Logistic if synth.SHAPES[name]["loss"] == "logistic" else LossKind.L2Svm
cfg = TrustRegionConfig(eps=0.01)
got = solve(p, loss, cfg, ExecutionPlan.gpu())
t1 = time.time()
w_ref, t_ref = Reference().solve(p, 0 if loss == LossKind.Logistic else 1, cfg, backend=Reference.PAR,
                                 workers=threads)
ref_s = time.time() - t1
out = {
    "workload": name, "threads": threads, "generate_s": gen_s, "reference_solve_s": ref_s,
    "objective": [got.objective, t_ref["objective"]],
    "rel_objective": abs(got.objective - t_ref["objective"]) / abs(t_ref["objective"]),
    "rel_w": float(np.linalg.norm(got.w - w_ref) / np.linalg.norm(w_ref)),
    "outer": [len(got.trace.iterations), len(t_ref["iterations"])],
    "accepted": [sum(it.accepted for it in got.trace.iterations), sum(it["accepted"] for it in t_ref["iterations"])],
    "cg_iters_gpu": [it.cg_iters for it in got.trace.iterations],
    "cg_iters_ref": [it["cg_iters"] for it in t_ref["iterations"]],
    "hv": [got.hessian_products, sum(it["cg_iters"] for it in t_ref["iterations"])],
}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"parity_{name}.json"), "w"), indent=1)
print(json.dumps(out))
