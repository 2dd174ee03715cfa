"""CPU tests: synthetic-input generator bit-exactness and multi-rank sharding (gloo, world size 2)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import reference as F
from oracle import restated as R
from paper_2409_15373_b200 import shard, synth


@pytest.mark.parametrize("kind,L,B,seed", [("uniform", 128, 64, 0), ("half-mean", 1024, 1024, 0),
                                           ("half-mean", 50, 33, 9), ("fixed", 7, 3, 1), ("uniform", 4096, 777, 5)])
def test_synth_lengths_bit_exact(kind, L, B, seed):
    got = synth.gen_lengths(kind, L, seed, B)
    np.testing.assert_array_equal(got, R.gen_lengths(kind, L, seed, B))
    if F.available():
        np.testing.assert_array_equal(got, F.gen_lengths(kind, L, seed, B))


@pytest.mark.parametrize("alpha,L,B", [(1.1, 512, 256), (0.8, 4096, 4096)])
def test_synth_zipf_bit_exact(alpha, L, B):
    np.testing.assert_array_equal(synth.gen_lengths("zipf", L, 0, B, alpha), R.gen_lengths("zipf", L, 0, B, alpha))


def test_synth_rng_stream():
    a, b = synth.Rng(123), R.Rng(123)
    for _ in range(1000):
        assert a.next_u64() == b.next_u64()


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_bounds_cover_and_balance(world):
    ln = synth.gen_lengths("half-mean", 1024, 0, 1024 * world)
    b = shard.shard_bounds(ln, world)
    assert b[0] == 0 and b[-1] == len(ln) and (np.diff(b) >= 0).all()
    cost = np.array([int((ln[b[k]:b[k + 1]] ** 2).sum()) for k in range(world)])
    assert abs(cost - cost.mean()).max() <= 1024 ** 2  # imbalance bounded by one sample
    rows = sum(shard.make_shard(ln, world, k).row_end - shard.make_shard(ln, world, k).row_begin for k in range(world))
    assert rows == ln.sum()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ln = synth.gen_lengths("half-mean", 1024, 0, 64 * world)
    sh = shard.make_shard(ln, world, rank)
    # each rank holds its contiguous value rows; gather them back and check the layout is bit-exact
    off = synth.offsets_of(ln)
    vals = torch.arange(int(off[-1]), dtype=torch.int64)[sh.row_begin:sh.row_end]
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([vals.numel()]))
    mx = int(max(s.item() for s in sizes))
    buf = torch.full((mx,), -1, dtype=torch.int64)
    buf[:vals.numel()] = vals
    outs = [torch.empty(mx, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(outs, buf)
    full = torch.cat([o[:int(s.item())] for o, s in zip(outs, sizes)])
    ok = bool(torch.equal(full, torch.arange(int(off[-1]))))
    rebased_ok = bool((sh.offsets == off[sh.sample_begin:sh.sample_end + 1] - off[sh.sample_begin]).all())
    # per-rank cost summed over ranks == total
    c = torch.tensor([int((sh.lengths ** 2).sum())])
    dist.all_reduce(c)
    q.put((rank, ok, rebased_ok, int(c.item()) == int((ln ** 2).sum())))
    dist.destroy_process_group()


def test_sharded_layout_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok and rb and tot for _, ok, rb, tot in res), res


def _mlp_worker(rank, world, port, q):
    """Each rank runs the (binary64) jagged_mlp_vjp on its sample shard; the all-reduced dW/db must equal the
    single-process gradients (the one op with a collective on its compute path)."""
    from oracle import restated as R

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ln = synth.gen_lengths("uniform", 40, 3, 16)
    off = synth.offsets_of(ln)
    rng = np.random.default_rng(7)
    dims = [6, 9, 4]
    layers = [(rng.uniform(-1, 1, (dims[l], dims[l + 1])), rng.uniform(-1, 1, dims[l + 1]), l == 0) for l in range(2)]
    x = rng.uniform(-1, 1, (int(off[-1]), dims[0]))
    go = rng.uniform(-1, 1, (int(off[-1]), dims[-1]))
    sh = shard.make_shard(ln, world, rank, cost="linear")
    _, g = R.jagged_mlp_vjp(x[sh.row_begin:sh.row_end], layers, go[sh.row_begin:sh.row_end])
    tg = [(torch.from_numpy(dw.copy()), torch.from_numpy(db.copy())) for dw, db in g]
    shard.all_reduce_mlp_grads(tg)
    _, full = R.jagged_mlp_vjp(x, layers, go)
    ok = all(np.allclose(a.numpy(), c, rtol=1e-12, atol=1e-12) and np.allclose(b.numpy(), d, rtol=1e-12, atol=1e-12)
             for (a, b), (c, d) in zip(tg, full))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_sharded_mlp_grads_allreduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_mlp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _scatter_worker(rank, world, port, q):
    """§8e setup + verification with gloo: rank 0 scatters a jagged batch on Bi^2-balanced boundaries, every
    rank runs the (binary64) attention oracle on its shard, rank 0 gathers outputs and lse rows back and
    compares with the single-process result (the computation shards with no collective)."""
    from oracle import restated as R

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ln = synth.gen_lengths("half-mean", 64, 5, 13)
    off = synth.offsets_of(ln)
    rows, D = int(off[-1]), 8
    full = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (rows, 3, D)))
    sh, local = shard.scatter_jagged(off if rank == 0 else None, full if rank == 0 else torch.empty(0, dtype=torch.float64),
                                     world, rank)
    o, lse = R.jfa_forward(sh.offsets, local[:, 0].numpy(), local[:, 1].numpy(), local[:, 2].numpy(), 64, 64)
    out = torch.cat([torch.from_numpy(o), torch.from_numpy(lse)[:, None]], 1)
    got = shard.gather_jagged(sh, out, off, world, rank)
    ok = True
    if rank == 0:
        ro, rl = R.jfa_forward(off, full[:, 0].numpy(), full[:, 1].numpy(), full[:, 2].numpy(), 64, 64)
        ok = np.allclose(got[:, :D].numpy(), ro, rtol=0, atol=0) and np.allclose(got[:, D].numpy(), rl, rtol=0, atol=0)
        ok = ok and torch.equal(local, full[sh.row_begin:sh.row_end])
    q.put((rank, bool(ok), sh.row_end - sh.row_begin))
    dist.destroy_process_group()


def test_scatter_compute_gather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_scatter_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(n > 0 for _, _, n in res), "both ranks hold rows"


def test_bench_gpus2_spawns_two_ranks():
    """`python bench.py --gpus 2` outside torchrun re-launches itself as two ranks (torch.distributed.run,
    rendezvous on 127.0.0.1); --selftest-launch exercises that plumbing on CPU (gloo all-reduce over the ranks)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest-launch"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert lines == [{"selftest": "launch", "n_ranks": 2, "rank_sum": 3.0, "backend": "gloo"}], p.stdout
