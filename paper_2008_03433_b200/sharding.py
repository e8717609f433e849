"""Row sharding of a problem across ranks.

Rank r of R owns the contiguous rows [l*r/R, l*(r+1)/R) of X and y; the
n-length vectors (w, g, d, p, M) are replicated.  Every per-rank
transposed product X_r^T u_r is a partial of the global one, summed by an
allreduce (NCCL on GPUs, gloo in the CPU tests) before the epilogue
``base + scale * sum``; every scalar sum (loss terms, |I|) likewise.  The
concatenation of the rank-local active sets in rank order is the global
ascending IndexSet.
"""
from __future__ import annotations

import numpy as np

from .tron import FeatureMatrix, Problem


def row_range(l: int, rank: int, world: int):
    return l * rank // world, l * (rank + 1) // world


def shard(problem: Problem, rank: int, world: int):
    """Returns (local problem, row_begin)."""
    X = problem.X
    b, e = row_range(X.rows, rank, world)
    if X.layout == "dense":
        vals = X.values.reshape(X.rows, X.cols)[b:e].reshape(-1)
        Xl = FeatureMatrix("dense", e - b, X.cols, np.ascontiguousarray(vals))
    else:
        s, t = X.row_offsets[b], X.row_offsets[e]
        ro = (X.row_offsets[b:e + 1] - s).astype(np.int64)
        Xl = FeatureMatrix("csr", e - b, X.cols, np.ascontiguousarray(X.values[s:t]), ro,
                           np.ascontiguousarray(X.col_indices[s:t]))
    return Problem(Xl, np.ascontiguousarray(problem.y[b:e]), problem.C), b


# ---------------------------------------------------------------------------
# Column partitioning
#
# Rank r owns the columns [n*r/R, n*(r+1)/R) of X -- its slice X_{:,r} kept as
# an l x n_r CSR (columns re-based to 0) plus its CSC -- and the matching
# slices of every n-vector (w, g, d, r, p, M).  The l-vectors (z, D, zhat, y,
# the SVM mask) are replicated.  Per call:
#   fun:  z = sum_r X_{:,r} w_r          l-length allreduce; loss terms local;
#         w.w = sum_r w_r.w_r            scalar allreduce
#   grad: g_r = w_r + C X_{:,r}^T zhat   local (no exchange); ||g||^2 scalar
#   Hv:   t = sum_r X_{:,r} v_r          l-length allreduce; a = D t;
#         out_r = v_r + C X_{:,r}^T a    local
#   CG:   p.Hp, r.z, r.r, ||d||^2, d.g, d.r  scalar allreduces
# so an Hv exchanges 8*l bytes instead of the row layout's 8*n (K1: 67 MB vs
# 160 MB; N1: 160 KB vs 10.8 MB).
# ---------------------------------------------------------------------------

def column_range(n: int, rank: int, world: int):
    return n * rank // world, n * (rank + 1) // world


def column_shard(problem: Problem, rank: int, world: int):
    """Returns (local problem l x n_r with columns re-based to 0, col_begin)."""
    X = problem.X
    b, e = column_range(X.cols, rank, world)
    if X.layout == "dense":
        vals = X.values.reshape(X.rows, X.cols)[:, b:e]
        Xl = FeatureMatrix("dense", X.rows, e - b, np.ascontiguousarray(vals).reshape(-1))
        return Problem(Xl, problem.y, problem.C), b
    ci = X.col_indices
    keep = (ci >= b) & (ci < e)
    rows = np.repeat(np.arange(X.rows), np.diff(X.row_offsets))
    counts = np.bincount(rows[keep], minlength=X.rows)
    ro = np.zeros(X.rows + 1, dtype=np.int64)
    np.cumsum(counts, out=ro[1:])
    Xl = FeatureMatrix("csr", X.rows, e - b, np.ascontiguousarray(X.values[keep]), ro,
                       np.ascontiguousarray((ci[keep] - b).astype(np.int32)))
    return Problem(Xl, problem.y, problem.C), b
