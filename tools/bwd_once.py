"""One cfg3 backward in each dQ mode (for ncu launch lists): python tools/bwd_once.py [det]"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

ln = synth.gen_lengths('half-mean', 1024, 0, 1024)
off = synth.offsets_of(ln)
S, H, D = int(off[-1]), 4, 128
mk = lambda: (torch.rand(S, H, D, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
T = lambda a: J.JaggedTensor(torch.from_numpy(off).cuda(), a, off)  # noqa: E731
Q, K, V, G = T(mk()), T(mk()), T(mk()), T(mk())
sch = J.Schedule(Q)
s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
for det in ([True, False] if len(sys.argv) < 2 else [sys.argv[1] == 'det']):
    J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch, deterministic=det)
torch.cuda.synchronize()
