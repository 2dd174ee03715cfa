"""Time one jagged op at the table1 shape (half-mean B=1024 L=1024 seed 0, D=T=128, bf16) — diagnostic, GPU only.

    python tools/op_bench.py jjjout|ajout|jd|jj|mlp [reps]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

op = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
B, L, D, T = 1024, 1024, 128, 128
ln = synth.gen_lengths("half-mean", L, 0, B)
off = synth.offsets_of(ln)
S, sq = int(off[-1]), int((ln * ln).sum())
offd = torch.from_numpy(off).cuda()
rnd = lambda *s: (torch.rand(*s, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
X, K2, Y = (J.JaggedTensor(offd, rnd(S, n), off) for n in (D, D, T))
A = J.Jagged2Tensor(offd, rnd(sq), off)
W = rnd(B, D, T)
layers = [J.MlpLayer(rnd(D, T), rnd(T), J.RELU), J.MlpLayer(rnd(T, D), rnd(D), J.NONE)]
fn = {"jjjout": lambda: J.jagged_jagged_bmm_jagged_out(X, K2), "ajout": lambda: J.array_jagged_bmm_jagged_out(A, X),
      "jd": lambda: J.jagged_dense_bmm(X, W), "jj": lambda: J.jagged_jagged_bmm(X, Y),
      "mlp": lambda: J.jagged_mlp(X, layers)}[op]
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
print(f"{op}: {np.median(ts) * 1e3:.1f} us (sum_sq={sq})")
