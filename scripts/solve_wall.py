"""Wall vs device time of repeated solves (host overhead per solve), device
loop on/off: python scripts/solve_wall.py R1 N1 ..."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, make_evaluator, synth

for W in sys.argv[1:] or ["R1", "N1"]:
    p = synth.make_shape(W)
    loss = LossKind.Logistic if synth.SHAPES[W]["loss"] == "logistic" else LossKind.L2Svm
    for loop in ("1", "0"):
        os.environ["TRON_B200_DEVICE_LOOP"] = loop
        with make_evaluator(p, loss, ExecutionPlan.gpu()) as ev:
            cfg = TrustRegionConfig(eps=0.01)
            for _ in range(3):
                ev.solve(cfg)
            wall, dev, call = [], [], []
            for _ in range(10):
                t0 = time.perf_counter()
                r = ev.solve(cfg)
                wall.append(time.perf_counter() - t0)
                dev.append(r.device_ms / 1e3)
            # the bare C call (no Python trace conversion)
            from paper_2008_03433_b200 import _lib
            import ctypes
            c = cfg.to_c()
            w = _lib.pinned_array(p.X.cols)
            tr = (_lib.tron_iteration * 1000)()
            info = _lib.tron_solve_info()
            for _ in range(10):
                t0 = time.perf_counter()
                _lib.lib.tron_gpu_solve(ev._h, ctypes.byref(c), None, w.ctypes.data_as(_lib.PD),
                                        ctypes.byref(info), tr, 1000)
                call.append(time.perf_counter() - t0)
        print(f"{W} device_loop={loop}: wall {np.median(wall)*1e3:.3f} ms, C call {np.median(call)*1e3:.3f} ms, "
              f"device {np.median(dev)*1e3:.3f} ms, outer {len(r.trace.iterations)} Hv {r.hessian_products}",
              flush=True)
