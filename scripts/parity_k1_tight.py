"""K1 parity against the reference at the bench eps and at a tight eps
("GPU and reference converge to the same optimum").

The reference solves come from scripts/ref_k1_local.py (the reference is
deterministic and thread-count independent, so they are the solves a run on
this box would produce); this script runs the GPU side on the same SYNTH-v1
input and writes gpurun_out/parity_K1.json in the format bench.py reads.
  python scripts/parity_k1_tight.py [tight_eps]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth  # noqa: E402

tight = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
scr = os.path.join(ROOT, "scratch")
refrec = json.load(open(os.path.join(scr, "k1_ref.json")))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def counts(res):
    its = res.trace.iterations
    return {"outer": len(its), "accepted": sum(1 for r in its if r.accepted),
            "cg_iters": [int(r.cg_iters) for r in its], "hv": int(res.hessian_products)}


t0 = time.time()
p = synth.make_shape("K1")
out = {"workload": "K1", "generator": "SYNTH-v1 seed 1", "generate_s": time.time() - t0,
       "reference_source": "scripts/ref_k1_local.py (unmodified reference, oracle/_ref; "
                           f"{refrec['threads']} threads; deterministic in the thread count)"}
with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
    sols = {}
    for e in (0.01, tight, 1e-8):
        r = ev.solve(TrustRegionConfig(eps=e))
        sols[e] = (r, r.w.copy())
res, w01 = sols[0.01]
rs = refrec["solves"]
r01 = rs["0.01"]
w_ref01 = np.load(os.path.join(scr, "k1_ref_0.01.npy"))
c = counts(res)
out["reference"] = {k: r01[k] for k in ("objective", "outer", "accepted", "cg_iters")}
out["reference"]["seconds"] = r01["seconds"]
par = {"rel_objective": abs(res.objective - r01["objective"]) / abs(r01["objective"]),
       "rel_w": rel(w01, w_ref01), "outer": [c["outer"], r01["outer"]],
       "accepted": [c["accepted"], r01["accepted"]], "cg_iters": [c["cg_iters"], r01["cg_iters"]],
       "hv": [c["hv"], sum(r01["cg_iters"])]}
par["gate_pass"] = bool(par["rel_objective"] <= 1e-6 and par["rel_w"] <= 1e-6
                        and all(abs(a - b) <= 1 for a, b in zip(*par["cg_iters"])))
w_star = sols[1e-8][1]
par["distance_to_optimum"] = {"optimum": "GPU solve at eps=1e-8", "rel_gpu": rel(w01, w_star),
                              "rel_reference": rel(w_ref01, w_star), "rel_between": par["rel_w"]}
par["both_meet_reference_stopping_rule"] = bool(
    r01["reference_gradient_norm_at_w"] <= 0.01 * r01["gradient_norm_initial"])
out["parity"] = par
key = repr(tight)
if key in rs:
    rt = rs[key]
    rr, wt = sols[tight]
    ct = counts(rr)
    w_reft = np.load(os.path.join(scr, f"k1_ref_{tight!r}.npy"))
    out["tight"] = {
        "eps": tight, "gpu": dict(objective=rr.objective, **ct),
        "reference": {k: rt[k] for k in ("objective", "outer", "accepted", "cg_iters", "seconds")},
        "rel_objective": abs(rr.objective - rt["objective"]) / abs(rt["objective"]),
        "rel_w": rel(wt, w_reft),
        "rel_w_gpu_to_optimum": rel(wt, w_star), "rel_w_reference_to_optimum": rel(w_reft, w_star),
    }
    out["tight"]["same_optimum"] = bool(out["tight"]["rel_objective"] <= 1e-10 and out["tight"]["rel_w"] <= 1e-6)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity_K1.json"), "w"), indent=1)
print(json.dumps(out))
