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


def scatter_jagged(offsets, values, world: int, rank: int, cost: str = "sq", src: int = 0, group=None):
    """SURVEY §8e setup: `src` holds the full jagged batch (host offsets [B+1] int64, values [rows, ...]); every
    rank receives its cost-balanced contiguous sample shard. Offsets go out by broadcast, each shard's rows by
    one point-to-point send (batched isend/irecv: NCCL over NVLink for CUDA tensors, gloo on CPU). Returns
    (Shard, local values). Non-src ranks pass values=None (CPU float32 receive buffers) or any tensor whose
    dtype/device the receive buffer should take."""
    import torch
    import torch.distributed as dist

    # control tensors live where the values do (NCCL moves CUDA tensors only; gloo CPU ones)
    dev = values.device if values is not None else torch.device("cpu")
    off_t = torch.as_tensor(np.asarray(offsets, np.int64)).to(dev) if rank == src else None
    n = torch.tensor([0 if off_t is None else off_t.numel()], dtype=torch.int64, device=dev)
    dist.broadcast(n, src, group=group)
    if off_t is None:
        off_t = torch.empty(int(n.item()), dtype=torch.int64, device=dev)
    dist.broadcast(off_t, src, group=group)
    off = off_t.cpu().numpy()
    sh = make_shard(np.diff(off), world, rank, cost)
    # row shape / dtype travel with a small header from src
    if rank == src:
        meta = torch.tensor([values.dim()] + list(values.shape[1:]) + [0] * (5 - values.dim()), dtype=torch.int64,
                            device=dev)
    else:
        meta = torch.empty(5, dtype=torch.int64, device=dev)
    dist.broadcast(meta, src, group=group)
    rest = [int(x) for x in meta[1:int(meta[0])].tolist()]
    bounds = shard_bounds(np.diff(off), world, cost)
    if rank == src:
        ops = []
        for r in range(world):
            r0, r1 = int(off[bounds[r]]), int(off[bounds[r + 1]])
            if r != src and r1 > r0:
                ops.append(dist.P2POp(dist.isend, values[r0:r1].contiguous(), r, group=group))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        local = values[sh.row_begin:sh.row_end].clone()
    else:
        local = torch.empty([sh.row_end - sh.row_begin] + rest, dtype=torch.float32 if values is None else values.dtype,
                            device="cpu" if values is None else values.device)
        if local.shape[0] > 0:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.irecv, local, src, group=group)]):
                w.wait()
    return sh, local


def gather_jagged(sh: Shard, local, offsets, world: int, rank: int, cost: str = "sq", dst: int = 0, group=None):
    """SURVEY §8e verification: the inverse of `scatter_jagged` — every rank's shard rows (outputs, grads, or lse
    rows) are sent to `dst`, which reassembles the full [rows, ...] tensor in sample order (None elsewhere)."""
    import torch
    import torch.distributed as dist

    off = np.asarray(offsets, np.int64)
    bounds = shard_bounds(np.diff(off), world, cost)
    if rank != dst:
        if local.shape[0] > 0:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(), dst, group=group)]):
                w.wait()
        return None
    full = torch.empty([int(off[-1])] + list(local.shape[1:]), dtype=local.dtype, device=local.device)
    ops = []
    for r in range(world):
        r0, r1 = int(off[bounds[r]]), int(off[bounds[r + 1]])
        if r == dst:
            full[r0:r1] = local
        elif r1 > r0:
            ops.append(dist.P2POp(dist.irecv, full[r0:r1], r, group=group))
    for w in dist.batch_isend_irecv(ops) if ops else []:
        w.wait()
    return full
