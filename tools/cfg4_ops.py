"""Run each cfg4 operator once (half-mean B=2048 L=1024 seed 0, D=T=256, bf16) — for ncu captures (diagnostic)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

ln = synth.gen_lengths("half-mean", 1024, 0, 2048)
off = synth.offsets_of(ln)
S, B, D, sq = int(off[-1]), len(ln), 256, int((ln * ln).sum())
offd = torch.from_numpy(off).cuda()
rnd = lambda *s: (torch.rand(*s, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
X, Y, GX = (J.JaggedTensor(offd, rnd(S, D), off) for _ in range(3))
A, GA = (J.Jagged2Tensor(offd, rnd(sq), off) for _ in range(2))
GZ = rnd(B, D, D)
ops = [lambda: J.jagged_jagged_bmm_jagged_out(X, Y), lambda: J.array_jagged_bmm_jagged_out(A, X),
       lambda: J.jagged_jagged_bmm(X, Y), lambda: J.jagged_softmax(X), lambda: J.jagged2_softmax(A),
       lambda: J.jagged_softmax_vjp(X, GX), lambda: J.jagged2_softmax_vjp(A, GA)]
for f in ops:
    f()
torch.cuda.synchronize()
