"""CPU, world_size 2 over gloo: the column-partitioned layout (SURVEY.md §8(f)
item 2; paper_2008_03433_b200.sharding.column_shard).

Rank r owns the columns [n r/R, n (r+1)/R) of X and the matching slices of the
n-vectors; the l-vectors are replicated.  An Hv exchanges one l-length
allreduce (t = sum_r X_{:,r} v_r) and the CG exchanges only scalars.  This
test is the executable specification of that schedule: each rank computes
its slice's partials with the oracle, the exchanges go through gloo, and

  * the composed fun / grad / Hv / preconditioner equal the unsharded ones;
  * a whole TRON-LR solve (tron.cpp:37-217) run in the column layout --
    CG with allreduced dots, the trust-region loop on the replicated
    scalars -- reproduces the oracle's solve: objective, w, every CG count.
"""
import math
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _log1p_exp_neg(t):  # loss.hpp:99-102
    return np.where(t >= 0.0, np.log1p(np.exp(-np.abs(t))), -t + np.log1p(np.exp(np.minimum(t, 0.0))))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    from paper_2008_03433_b200 import TrustRegionConfig, synth
    from paper_2008_03433_b200.sharding import column_range, column_shard
    from pyoracle import Port
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_ = Port()

    def allreduce(x):
        t = torch.from_numpy(np.array(x, dtype=np.float64, copy=True).reshape(-1))
        dist.all_reduce(t)
        return t.numpy()

    def gdot(a, b):  # a CG dot over column-partitioned vectors: one scalar allreduce
        return float(allreduce([float(a @ b)])[0])

    try:
        out = {}
        p = synth.synth_sparse(11, 900, 6000, 25)
        loc, c0 = column_shard(p, rank, world)
        b, e = column_range(p.X.cols, rank, world)
        assert (c0, c0 + loc.X.cols) == (b, e)
        y, C, n = p.y, p.C, p.X.cols

        def rowdots(v_r):  # X_{:,r} v_r (partial, l-length)
            return port_.logistic(loc, v_r)["z"]

        def fun(w_r):  # fused pass in the column layout
            z = allreduce(rowdots(w_r))                      # l-length exchange
            t = y * z
            sig = 1.0 / (1.0 + np.exp(t))
            zhat, dvec = -y * sig, (1.0 - sig) * sig
            ww = gdot(w_r, w_r)                               # scalar exchange
            return 0.5 * ww + C * float(np.sum(_log1p_exp_neg(t))), zhat, dvec

        def grad(w_r, zhat):  # local: no exchange
            return w_r + C * port_.matvec_transpose(loc.X, zhat)

        def hv(v_r, dvec):
            tvec = allreduce(rowdots(v_r))                     # l-length exchange
            return v_r + C * port_.matvec_transpose(loc.X, dvec * tvec)

        # ---- composed evaluator at a fixed point
        w = synth.testgen_random_vector(5, n, 0.3)
        v = synth.testgen_random_vector(6, n)
        f, zhat, dvec = fun(w[b:e])
        g_r = grad(w[b:e], zhat)
        hv_r = hv(v[b:e], dvec)
        sq = loc.X.__class__("csr", loc.X.rows, loc.X.cols, loc.X.values ** 2, loc.X.row_offsets,
                             loc.X.col_indices)
        m_r = 1.0 + C * port_.matvec_transpose(sq, dvec)
        parts = [None] * world
        dist.all_gather_object(parts, (g_r.tolist(), hv_r.tolist(), m_r.tolist()))
        out["f"] = f
        out["g"] = sum((x[0] for x in parts), [])
        out["hv"] = sum((x[1] for x in parts), [])
        out["M"] = sum((x[2] for x in parts), [])

        # ---- a whole TRON solve in the column layout (tron.cpp:37-217)
        cfg = TrustRegionConfig(eps=1e-3)
        max_cg = min(n, 1000)
        w_r = np.zeros(e - b)
        f, zhat, dvec = fun(w_r)
        g_r = grad(w_r, zhat)
        gnorm0 = math.sqrt(gdot(g_r, g_r))
        gnorm, delta, cg_counts = gnorm0, gnorm0, []
        while len(cg_counts) < cfg.max_outer_iters and gnorm > cfg.eps * gnorm0:
            d = np.zeros_like(w_r)
            r = -g_r
            pv = r.copy()
            rz = gdot(r, r)
            stop = cfg.cg_tol * gnorm
            it = 0
            while it < max_cg:
                if math.sqrt(gdot(r, r)) <= stop:
                    break
                it += 1
                hp = hv(pv, dvec)
                alpha = rz / gdot(pv, hp)
                d = d + alpha * pv
                if math.sqrt(gdot(d, d)) > delta:
                    d = d - alpha * pv
                    dp, dd, pp = gdot(d, pv), gdot(d, d), gdot(pv, pv)
                    rad = math.sqrt(dp * dp + pp * (delta * delta - dd))
                    tau = (delta * delta - dd) / (dp + rad) if dp >= 0.0 else (rad - dp) / pp
                    d = d + tau * pv
                    r = r - tau * hp
                    break
                r = r - alpha * hp
                rz_next = gdot(r, r)
                pv = r + (rz_next / rz) * pv
                rz = rz_next
            q_model = 0.5 * (gdot(d, g_r) - gdot(d, r))
            step = math.sqrt(gdot(d, d))
            f_c, zhat_c, dvec_c = fun(w_r + d)
            sigma = (f_c - f) / q_model
            accept = sigma > cfg.sigma0
            if not accept:
                delta = cfg.gamma1 * step
            elif sigma < cfg.eta1:
                delta = cfg.gamma2 * step
            elif sigma >= cfg.eta2:
                delta = max(cfg.gamma3 * step, delta)
            cg_counts.append(it)
            if accept:
                w_r, f, zhat, dvec = w_r + d, f_c, zhat_c, dvec_c
                g_r = grad(w_r, zhat)
                gnorm = math.sqrt(gdot(g_r, g_r))
        ws = [None] * world
        dist.all_gather_object(ws, w_r.tolist())
        out["solve"] = dict(w=sum(ws, []), f=f, cg=cg_counts)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_column_partition_composes(port):
    from paper_2008_03433_b200 import TrustRegionConfig, synth
    from pyoracle import LOGISTIC
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pt = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, pt, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = synth.synth_sparse(11, 900, 6000, 25)
    n = p.X.cols
    w = synth.testgen_random_vector(5, n, 0.3)
    v = synth.testgen_random_vector(6, n)
    full = port.logistic(p, w, v)
    assert abs(out["f"] - full["f"]) <= 1e-12 * abs(full["f"])
    for k in ("g", "hv", "M"):
        assert np.allclose(out[k], full[k], rtol=1e-12, atol=1e-13), k
    w_ref, t_ref = port.solve(p, LOGISTIC, TrustRegionConfig(eps=1e-3))
    got = out["solve"]
    assert abs(got["f"] - t_ref["objective"]) <= 1e-10 * abs(t_ref["objective"])
    assert np.linalg.norm(np.array(got["w"]) - w_ref) <= 1e-8 * np.linalg.norm(w_ref)
    assert got["cg"] == [it["cg_iters"] for it in t_ref["iterations"]]
