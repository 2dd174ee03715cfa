"""Batch sharding across GPUs on cost-balanced sample boundaries.

Every hot-path op computes sample i from sample i's rows only (linalg.cpp:47-66,
attention.cpp:186-289), so ranks take contiguous sample ranges [b_k, b_{k+1}) and need no
collective on the compute path. Boundaries split the prefix sum of per-sample cost — Bi^2 for
attention and the jagged_out ops, Bi for the linear ops — so imbalance is at most one sample.
A shard's values are the contiguous row range [offsets[b_k], offsets[b_{k+1}]) and its offsets are
rebased by -offsets[b_k] (integer, bit-exact).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_bounds(lengths, world: int, cost: str = "sq") -> np.ndarray:
    ln = np.asarray(lengths, np.int64)
    c = ln * ln if cost == "sq" else ln.copy()
    pre = np.concatenate([[0], np.cumsum(c)])
    total = pre[-1]
    bounds = [0]
    for k in range(1, world):
        target = total * k / world
        # first boundary whose prefix reaches the target, never before the previous boundary
        b = int(np.searchsorted(pre, target, side="left"))
        if b > 0 and abs(pre[b - 1] - target) <= abs(pre[b] - target):
            b -= 1
        bounds.append(max(b, bounds[-1]))
    bounds.append(len(ln))
    return np.asarray(bounds, np.int64)


@dataclass
class Shard:
    rank: int
    sample_begin: int
    sample_end: int
    row_begin: int
    row_end: int
    offsets: np.ndarray  # rebased, [n_samples + 1]

    @property
    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)


def make_shard(lengths, world: int, rank: int, cost: str = "sq") -> Shard:
    ln = np.asarray(lengths, np.int64)
    b = shard_bounds(ln, world, cost)
    off = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
    s0, s1 = int(b[rank]), int(b[rank + 1])
    return Shard(rank, s0, s1, int(off[s0]), int(off[s1]), off[s0:s1 + 1] - off[s0])


def all_reduce_mlp_grads(dlayers, group=None) -> None:
    """jagged_mlp_vjp under sample sharding: dW and db are sums over all rows
    (linalg.cpp:540-554), so each rank's shard gives a partial sum; one in-place SUM all-reduce per
    tensor (NCCL over NVLink for CUDA tensors, gloo on CPU) makes them the full-batch gradients.
    dx stays per-rank (rows are not shared). `dlayers`: objects with .dweights/.dbias or (dW, db) pairs."""
    import torch.distributed as dist

    for g in dlayers:
        for t in ((g.dweights, g.dbias) if hasattr(g, "dweights") else g):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
