"""Host-side overhead of GpuEvaluator.solve (w download, result marshalling) for a shape."""
import ctypes, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth, _lib
from paper_2008_03433_b200._lib import lib
name = sys.argv[1] if len(sys.argv) > 1 else "N1"
p = synth.make_shape(name)
cfg = TrustRegionConfig(eps=0.01)
with make_evaluator(p, LossKind.Logistic, ExecutionPlan.gpu()) as ev:
    ev.solve(cfg)
    for kind in ("zeros", "empty", "reused", "pinned"):
        pinned = torch.empty(p.X.cols, dtype=torch.float64, pin_memory=True).numpy()
        reused = np.zeros(p.X.cols); reused[:] = 1.0
        ts = []
        for _ in range(5):
            c = cfg.to_c(_lib.SOLVE_DEVICE)
            info = _lib.tron_solve_info()
            w = {"zeros": lambda: np.zeros(p.X.cols), "empty": lambda: np.empty(p.X.cols),
                 "reused": lambda: reused, "pinned": lambda: pinned}[kind]()
            t0 = time.perf_counter()
            lib.tron_gpu_solve(ev._h, ctypes.byref(c), None, w.ctypes.data_as(_lib.PD), ctypes.byref(info), None, 0)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name} w={kind}: C solve call {min(ts):.2f} ms (device {info.device_ms:.2f})", flush=True)
    t0 = time.perf_counter(); ev.solve(cfg); print(f"{name} Python ev.solve {1e3*(time.perf_counter()-t0):.2f} ms")
