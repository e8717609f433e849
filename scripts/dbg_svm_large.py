import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, solve, synth, SvmStrategy
from pyoracle import Reference
ref = Reference()
p = synth.synth_sparse(11, 6000, 300_000, 30)
cfg = TrustRegionConfig(eps=0.01)
w_ref, t_ref = ref.solve(p, 1, cfg, backend=1, workers=8)
print("ref", t_ref["objective"], [(it["cg_iters"], it["accepted"]) for it in t_ref["iterations"]])
for env in ({}, {"TRON_B200_COOP_CG": "0"}, {"TRON_B200_NO_GRAPH": "1"}):
    for k in ("TRON_B200_COOP_CG", "TRON_B200_NO_GRAPH"): os.environ.pop(k, None)
    os.environ.update(env)
    r = solve(p, LossKind.L2Svm, cfg, ExecutionPlan.gpu(svm_strategy=SvmStrategy.Indirect))
    print(env, r.objective, np.linalg.norm(r.w - w_ref) / np.linalg.norm(w_ref),
          [(it.cg_iters, it.accepted) for it in r.trace.iterations])
