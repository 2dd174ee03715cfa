"""Time the tcgen05 attention kernels over several length distributions (diagnostic, GPU only).

Usage: python tools/attn_sweep.py   — prints one line per distribution with fwd/bwd ms and TF/s.
Long uniform samples isolate the per-block pipeline; short ones expose per-item (K/V reload,
dK/dV epilogue) overhead.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

DET = os.environ.get('JG_SWEEP_DET', '1') != '0'  # backward dQ accumulation mode


def run(name, ln, H=4, D=128, reps=25):
    off = synth.offsets_of(ln)
    S = int(off[-1])
    mk = lambda: (torch.rand(S, H, D, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).cuda(), a, off)  # noqa: E731
    Q, K, V, G = T(mk()), T(mk()), T(mk()), T(mk())
    sch = J.Schedule(Q)
    for _ in range(3):
        s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
        J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch, deterministic=DET)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tfs, tbs = [], []
    for _ in range(reps):
        ev[0].record()
        s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
        ev[1].record()
        J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch, deterministic=DET)
        ev[2].record()
        torch.cuda.synchronize()
        tfs.append(ev[0].elapsed_time(ev[1]))
        tbs.append(ev[1].elapsed_time(ev[2]))
    tf, tb = float(np.median(tfs)), float(np.median(tbs))  # median: robust to clock/thermal noise
    sq = float((np.asarray(ln, np.float64) ** 2).sum())
    ff, fb = 4 * sq * H * D, 10 * sq * H * D
    print(f"{name:24s} sumB={S:8d} fwd {tf:7.3f} ms {ff / tf / 1e9:7.1f} TF/s   bwd {tb:7.3f} ms {fb / tb / 1e9:7.1f} TF/s",
          flush=True)


if __name__ == '__main__':
    run('half-mean B1024 L1024', synth.gen_lengths('half-mean', 1024, 0, 1024))
    run('uniform-full B512 L1024', np.full(512, 1024, np.int64))
    run('full B128 L2048', np.full(128, 2048, np.int64))
    run('full B32 L4096', np.full(32, 4096, np.int64))
    run('full B2048 L256', np.full(2048, 256, np.int64))
