import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, solve, synth
cfg = TrustRegionConfig(eps=0.01)
cases = {"svm_20000x40": (synth.synth_dense(1, 20000, 40), LossKind.L2Svm),
         "lr_20000x40": (synth.synth_dense(1, 20000, 40), LossKind.Logistic),
         "svm_200x20": (synth.testgen_dense_problem(3001, 200, 20, 1.0), LossKind.L2Svm)}
for name, (p, loss) in cases.items():
    os.environ["TRON_B200_FORCE_NCCL"] = "0"
    a = solve(p, loss, cfg, ExecutionPlan.gpu())
    os.environ["TRON_B200_FORCE_NCCL"] = "1"
    b = solve(p, loss, cfg, ExecutionPlan.gpu())
    os.environ["TRON_B200_FORCE_NCCL"] = "0"
    os.environ["TRON_B200_NO_GRAPH"] = "1"
    c = solve(p, loss, cfg, ExecutionPlan.gpu())
    del os.environ["TRON_B200_NO_GRAPH"]
    print(name, a.objective, b.objective, c.objective, [it.cg_iters for it in a.trace.iterations],
          [it.cg_iters for it in b.trace.iterations], [it.cg_iters for it in c.trace.iterations], flush=True)
