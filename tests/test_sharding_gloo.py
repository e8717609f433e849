"""CPU, world_size 2 over gloo: the row-sharded composition the multi-GPU
path uses (paper_2008_03433_b200.sharding; engine.cpp allreduces the same
partials over NCCL).  Each rank computes its shard's partials with the
oracle; after an allreduce they must reproduce the unsharded fun / grad /
Hv / preconditioner, and the rank-ordered concatenation of local active sets
must be the global ascending IndexSet."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    from paper_2008_03433_b200 import synth
    from paper_2008_03433_b200.sharding import row_range, shard
    from pyoracle import Port
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port_ = Port()
        out = {}
        for name, p in (("sparse", synth.testgen_sparse_problem(77, 301, 40, 1.5, 0.2)),
                        ("dense", synth.synth_dense(3, 997, 12))):
            loc, b = shard(p, rank, world)
            assert (b, b + loc.X.rows) == row_range(p.X.rows, rank, world)
            n = p.X.cols
            w = synth.testgen_random_vector(5, n, 0.3)
            v = synth.testgen_random_vector(6, n)
            # raw per-shard partials: transposed products with base 0, scale 1
            lr = port_.logistic(loc, w, v)
            zero = np.zeros(n)
            part = {
                "loss": float(np.sum(lr["alpha"])),
                "g": port_.matvec_transpose(loc.X, lr["zhat"]),
                "hv": port_.matvec_transpose(loc.X, _dv(port_, loc, v) * lr["dvec"]),
                "M": port_.matvec_transpose(_sq(loc.X), lr["dvec"]),
            }
            for k in ("g", "hv", "M"):
                t = torch.from_numpy(part[k].copy())
                dist.all_reduce(t)
                part[k] = t.numpy()
            t = torch.tensor([part["loss"]], dtype=torch.float64)
            dist.all_reduce(t)
            sv = port_.svm(loc, w, zero)
            act = [None] * world
            dist.all_gather_object(act, (sv["active"] + b).tolist())
            out[name] = dict(f=0.5 * float(w @ w) + p.C * float(t[0]),
                             g=w + p.C * part["g"], hv=v + p.C * part["hv"],
                             M=1.0 + p.C * part["M"], active=sum(act, []))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _dv(port_, loc, v):
    from paper_2008_03433_b200.tron import FeatureMatrix  # noqa: F401
    return loc.X.to_dense() @ v


def _sq(X):
    from paper_2008_03433_b200.tron import FeatureMatrix
    if X.layout == "dense":
        return FeatureMatrix("dense", X.rows, X.cols, X.values * X.values)
    return FeatureMatrix("csr", X.rows, X.cols, X.values * X.values, X.row_offsets, X.col_indices)


def test_two_rank_sharded_partials_compose(port):
    from paper_2008_03433_b200 import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, p_, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for name, p in (("sparse", synth.testgen_sparse_problem(77, 301, 40, 1.5, 0.2)),
                    ("dense", synth.synth_dense(3, 997, 12))):
        n = p.X.cols
        w = synth.testgen_random_vector(5, n, 0.3)
        v = synth.testgen_random_vector(6, n)
        full = port.logistic(p, w, v)
        got = out[name]
        assert abs(got["f"] - full["f"]) <= 1e-12 * abs(full["f"])
        for k in ("g", "hv", "M"):
            assert np.allclose(got[k], full[k], rtol=1e-12, atol=1e-12), (name, k)
        sv = port.svm(p, w, np.zeros(n))
        assert got["active"] == sv["active"].tolist()
