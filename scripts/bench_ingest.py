"""Ingestion benchmark: LIBSVM text of a SYNTH-v1 shape
parsed by the native parallel parser vs the reference's parse_libsvm (oracle/_ref,
single-threaded istream), and file -> trained model through the public API.
Usage: python scripts/bench_ingest.py [N1]   (writes gpurun_out/ingest_<W>.json)"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2008_03433_b200 import ExecutionPlan, LossKind, TrustRegionConfig, io, solve, synth
from pyoracle import Reference

name = sys.argv[1] if len(sys.argv) > 1 else "N1"
p = synth.make_shape(name)
t0 = time.perf_counter()
text = io.write_libsvm(p)
write_s = time.perf_counter() - t0
path = os.path.join("/tmp", f"tron_{name}.svm")
with open(path, "wb") as f:
    f.write(text)
mb = len(text) / 1e6

def best(fn, reps):
    ts = []
    for _ in range(reps):
        t = time.perf_counter(); r = fn(); ts.append(time.perf_counter() - t)
    return min(ts), r

t_mem, q = best(lambda: io.parse_libsvm(text), 5)
t_file, _ = best(lambda: io.parse_libsvm(path), 5)
ref = Reference()
t_ref, (kind, arrays) = best(lambda: ref.parse_libsvm(text), 2)
same = kind == "ok" and np.array_equal(arrays[2].view(np.uint64), q.X.values.view(np.uint64)) \
    and np.array_equal(arrays[1], q.X.col_indices) and np.array_equal(arrays[0], q.X.row_offsets)
cfg = TrustRegionConfig(eps=0.01)
loss = LossKind.Logistic if synth.SHAPES[name]["loss"] == "logistic" else LossKind.L2Svm
solve(io.parse_libsvm(path), loss, cfg, ExecutionPlan.gpu())  # warm
t_e2e, r = best(lambda: solve(io.parse_libsvm(path), loss, cfg, ExecutionPlan.gpu()), 3)
out = {"workload": name, "text_mb": mb, "host_cores": len(os.sched_getaffinity(0)),
       "native_parse_bytes_s": t_mem, "native_parse_file_s": t_file, "reference_parse_s": t_ref,
       "native_mb_per_s": mb / t_mem, "reference_mb_per_s": mb / t_ref, "speedup": t_ref / t_mem,
       "identical_to_reference": bool(same), "file_to_model_s": t_e2e, "objective": r.objective}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"ingest_{name}.json"), "w"), indent=1)
print(json.dumps(out))
