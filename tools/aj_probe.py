"""array_jagged_bmm_jagged_out at the cfg4 shape (half-mean B=2048 L=1024 seed 0, D=256, bf16) — diagnostic, GPU
only: median time of the op (and of its VJP with `vjp`) for ncu captures and A/B runs."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
what = sys.argv[2] if len(sys.argv) > 2 else "fwd"
ln = synth.gen_lengths("half-mean", 1024, 0, 2048)
off = synth.offsets_of(ln)
S, D, sq = int(off[-1]), 256, int((ln * ln).sum())
offd = torch.from_numpy(off).cuda()
rnd = lambda *s: (torch.rand(*s, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
X, GX = (J.JaggedTensor(offd, rnd(S, D), off) for _ in range(2))
A = J.Jagged2Tensor(offd, rnd(sq), off)
fn = {"fwd": lambda: J.array_jagged_bmm_jagged_out(A, X),
      "vjp": lambda: J.array_jagged_bmm_jagged_out_vjp(A, X, GX),
      "jjj": lambda: J.jagged_jagged_bmm_jagged_out(X, GX)}[what]
for _ in range(2):
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
byts = (2 * S * D + sq) * 2
print(f"{what}: {np.median(ts) * 1e3:.1f} us  {byts / np.median(ts) / 1e6:.0f} GB/s (fwd bytes)")
