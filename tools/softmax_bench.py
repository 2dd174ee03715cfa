"""Time the jagged softmax kernels at the cfg4 shape (half-mean B=2048 L=1024 seed 0, sum_B = 1,048,576, D = 256,
bf16) — diagnostic, GPU only. Prints ms and GB/s (algorithmic bytes: read x (+ g) + write out).

    python tools/softmax_bench.py [reps]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ln = synth.gen_lengths("half-mean", 1024, 0, 2048)
off = synth.offsets_of(ln)
S, D, sq = int(off[-1]), 256, int((ln * ln).sum())
offd = torch.from_numpy(off).cuda()
rnd = lambda *s: (torch.rand(*s, device='cuda') * 8 - 4).bfloat16()  # noqa: E731
X, GX = (J.JaggedTensor(offd, rnd(S, D), off) for _ in range(2))
A, GA = (J.Jagged2Tensor(offd, rnd(sq), off) for _ in range(2))
ops = {"jagged_softmax": (lambda: J.jagged_softmax(X), 2 * S * D * 2),
       "jagged_softmax_vjp": (lambda: J.jagged_softmax_vjp(X, GX), 3 * S * D * 2),
       "jagged2_softmax": (lambda: J.jagged2_softmax(A), 2 * sq * 2),
       "jagged2_softmax_vjp": (lambda: J.jagged2_softmax_vjp(A, GA), 3 * sq * 2)}
for name, (fn, byts) in ops.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"{name:22s} {ms * 1e3:8.1f} us  {byts / ms / 1e6:8.1f} GB/s", flush=True)
