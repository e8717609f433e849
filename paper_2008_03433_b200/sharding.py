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
