"""Objective / counts of one dense L2-SVM solve under every Gram mode and the reference."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
from pyoracle import Reference
p = synth.synth_dense(1, 200_000, 40)
eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
cfg = TrustRegionConfig(eps=eps)
modes = {"delta": {}, "fresh": {"TRON_B200_GRAM_DELTA": "0"}, "fused": {"TRON_B200_GRAM_FUSED": "1"},
         "traversal": {"TRON_B200_DENSE_GRAM": "0"}}
ws = {}
for name, env in modes.items():
    for k in ("TRON_B200_GRAM_DELTA", "TRON_B200_GRAM_FUSED", "TRON_B200_DENSE_GRAM"):
        os.environ.pop(k, None)
    os.environ.update(env)
    with make_evaluator(p, LossKind.L2Svm, ExecutionPlan.gpu()) as ev:
        r = ev.solve(cfg)
    ws[name] = r.w
    print(json.dumps({"mode": name, "f": r.objective, "cg": [it.cg_iters for it in r.trace.iterations],
                      "f_seq": [it.f_candidate for it in r.trace.iterations]}))
w_ref, t_ref = Reference().solve(p, 1, cfg)
print(json.dumps({"mode": "reference", "f": t_ref["objective"], "cg": [it["cg_iters"] for it in t_ref["iterations"]],
                  "f_seq": [it.get("f_candidate") for it in t_ref["iterations"]]}))
for k, w in ws.items():
    print(k, "rel_w vs ref", float(np.linalg.norm(w - w_ref) / np.linalg.norm(w_ref)))
