import os, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth
ln = (np.full(2048, int(sys.argv[1]), np.int64) if len(sys.argv) > 1 else synth.gen_lengths('half-mean', 1024, 0, 1024)); off = synth.offsets_of(ln); S = int(off[-1]); H, D = 4, 128
mk = lambda: (torch.rand(S, H, D, device='cuda') * 2 - 1).bfloat16()
T = lambda a: J.JaggedTensor(torch.from_numpy(off).cuda(), a, off)
Q, K, V, G = T(mk()), T(mk()), T(mk()), T(mk())
sch = J.Schedule(Q)
for _ in range(2):
    s = J.jagged_flash_attention_forward(Q, K, V, schedule=sch)
    J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sch, deterministic=os.environ.get('JG_SWEEP_DET', '1') != '0')
torch.cuda.synchronize()
