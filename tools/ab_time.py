"""A/B timing of the attention kernels for the library JG_LIB_PATH points at (diagnostic, GPU only).

    JG_LIB_PATH=abtest/<name>/libjagged_b200.so python tools/ab_time.py [tag]
Prints median fwd / bwd ms on cfg3 (half-mean B=1024 L=1024 H=4 D=128) and on uniform L=4096.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402


def run(name, ln, H=4, D=128, reps=20):
    off = synth.offsets_of(ln)
    S = int(off[-1])
    g = torch.Generator(device='cuda').manual_seed(0)
    mk = lambda: (torch.rand(S, H, D, device='cuda', generator=g) * 2 - 1).bfloat16()  # noqa: E731
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).cuda(), a, off)  # noqa: E731
    Q, K, V, G = T(mk()), T(mk()), T(mk()), T(mk())
    sch = J.Schedule(Q)
    for _ in range(3):
        s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
        J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(reps):
        ev[0].record()
        s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
        ev[1].record()
        gr = J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch)
        ev[2].record()
        torch.cuda.synchronize()
        tf.append(ev[0].elapsed_time(ev[1]))
        tb.append(ev[1].elapsed_time(ev[2]))
    ck = float(gr.dq.values.float().abs().sum() + gr.dk.values.float().abs().sum() + gr.dv.values.float().abs().sum())
    sq = float((np.asarray(ln, np.float64) ** 2).sum())
    mb = float(np.median(tb))
    print(f"{sys.argv[1] if len(sys.argv) > 1 else '':10s} {name:12s} fwd {np.median(tf):6.3f} ms  bwd {mb:6.3f} ms "
          f"{10 * sq * H * D / mb / 1e9:6.1f} TF/s  checksum {ck:.6e}", flush=True)


if __name__ == '__main__':
    run('cfg3', synth.gen_lengths('half-mean', 1024, 0, 1024))
    run('L4096', np.full(32, 4096, np.int64))
