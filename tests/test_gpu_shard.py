"""bench.py's sharded verification leg on the device: scatter a verification batch over NCCL,
fwd+bwd per shard, gather outputs / lse / grads back and compare with the unsharded run bit for bit. One GPU is
available here, so the NCCL group has one rank (the code path is the same; the multi-rank plumbing is covered
on CPU/gloo by tests/test_synth_shard.py)."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_verify_leg_nccl_world1():
    import torch.distributed as dist

    import bench

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(bench._free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        v = bench.verify_sharded(1, 0, torch.device("cuda", 0), n_samples=48)
    finally:
        dist.destroy_process_group()
    assert v["bit_identical"] and v["unsharded_match"] and v["collective"] == "nccl" and v["samples"] == 48
