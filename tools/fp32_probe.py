"""fp32-mode jagged flash attention timing (diagnostic, GPU only): cfg3 lengths (half-mean B=1024 L=1024),
H=4, D=128, fp32 in/out; the reference's own float API reaches this path through the C++ drop-in.
Usage: fp32_probe.py [B] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ln = synth.gen_lengths('half-mean', 1024, 0, B)
off = synth.offsets_of(ln)
S, H, D = int(off[-1]), 4, 128
mk = lambda: (torch.rand(S, H, D, device='cuda') * 2 - 1)  # noqa: E731
T = lambda a: J.JaggedTensor(torch.from_numpy(off).cuda(), a, off)  # noqa: E731
Q, K, V, G = T(mk()), T(mk()), T(mk()), T(mk())
sch = J.Schedule(Q)
s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch)
torch.cuda.synchronize()
sq = float((ln.astype(np.float64) ** 2).sum())
for _ in range(reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
    ev[1].record()
    J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch)
    ev[2].record()
    torch.cuda.synchronize()
    tf, tb = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    print(f"fp32 B={B}: fwd {tf:.2f} ms ({4 * sq * H * D / tf / 1e9:.2f} TF/s)  "
          f"bwd {tb:.2f} ms ({10 * sq * H * D / tb / 1e9:.2f} TF/s)")
