"""Time feature_interaction (bf16): the fused cross-attention kernel vs the composed path (JG_ATTN_IMPL=simt).

    python tools/fi_bench.py            — half-mean B=1024 L=1024 seed 0 keys, D=128, Tq=64 targets per sample
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

B, L, D, Tq = 1024, 1024, 128, 64
ln = synth.gen_lengths("half-mean", L, 0, B)
off = synth.offsets_of(ln)
S = int(off[-1])
offd = torch.from_numpy(off).cuda()
r = lambda *s: (torch.rand(*s, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
K, V = J.JaggedTensor(offd, r(S, D), off), J.JaggedTensor(offd, r(S, D), off)
T = r(B, Tq, D)
fn = lambda: J.feature_interaction(K, V, T)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
fl = 4.0 * S * Tq * D
print(f"feature_interaction B={B} L={L} D={D} Tq={Tq}: {ms * 1e3:.1f} us, {fl / ms / 1e9:.1f} TFLOP/s")
