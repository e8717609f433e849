import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, solve, synth
p = synth.synth_sparse(9, 2000, 5000, 37)
cfg = TrustRegionConfig(eps=0.01)
def run(env):
    for k in ("TRON_B200_NO_GRAPH", "TRON_B200_FORCE_NCCL", "TRON_B200_NCCL_GRAPH"):
        os.environ.pop(k, None)
    os.environ.update(env)
    r = solve(p, LossKind.Logistic, cfg, ExecutionPlan.gpu())
    return r.objective.hex(), [it.cg_iters for it in r.trace.iterations], r.w
outs = {}
for name, env in [("nograph", {"TRON_B200_NO_GRAPH": "1"}), ("nograph2", {"TRON_B200_NO_GRAPH": "1"}),
                  ("graph", {}), ("nccl_host", {"TRON_B200_FORCE_NCCL": "1", "TRON_B200_NCCL_GRAPH": "0"}),
                  ("nccl_host2", {"TRON_B200_FORCE_NCCL": "1", "TRON_B200_NCCL_GRAPH": "0"})]:
    outs[name] = run(env)
    f, it, w = outs[name]
    print(name, f, it, np.abs(w - outs["nograph"][2]).max())
