"""Wall vs device time of consecutive solves (diagnoses per-step outliers)."""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth
W = sys.argv[1] if len(sys.argv) > 1 else "R1"
mode = sys.argv[2] if len(sys.argv) > 2 else "evict"
p = synth.make_shape(W)
loss = LossKind.Logistic if synth.SHAPES[W]["loss"] == "logistic" else LossKind.L2Svm
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cfg = TrustRegionConfig(eps=0.01)
with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
    for _ in range(int(os.environ.get("WARM", "3"))):
        ev.solve(cfg)
    walls, devs = [], []
    gc.disable()
    for k in range(int(os.environ.get("STEPS", "12"))):
        if mode == "evict":
            flush.view(torch.int64).sum()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ev.solve(cfg)
        walls.append(round((time.perf_counter() - t0) * 1e3, 3))
        devs.append(round(r.device_ms, 3))
    gc.enable()
print(W, mode, "wall", walls)
print(W, mode, "dev ", devs)
