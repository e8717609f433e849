"""Standalone N1 Hv/grad/fun launches for ncu (kernels replayed by the profiler)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, make_evaluator, synth
name = sys.argv[1] if len(sys.argv) > 1 else "N1"
p = synth.make_shape(name)
loss = LossKind.Logistic if synth.SHAPES[name]["loss"] == "logistic" else LossKind.L2Svm
with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
    ev.eval_candidate(np.zeros(p.X.cols)); ev.commit()
    print(ev.bench_kernels(reps=3, flush_l2=True))
