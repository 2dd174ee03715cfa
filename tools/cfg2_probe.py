"""cfg2 forward probe (diagnostic, GPU only): eager and CUDA-graph times of the JFA forward on the cfg2 workload
(Zipf(1.1) B=256 L=512 D=64 H=1 bf16), for ncu launch lists."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth  # noqa: E402

ln = synth.gen_lengths("zipf", 512, 0, 256, 1.1)
off = synth.offsets_of(ln)
S, D, H = int(off[-1]), 64, 1
mk = lambda: (torch.rand(S, H, D, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
Q, K, V = (J.JaggedTensor(torch.from_numpy(off).cuda(), mk(), off) for _ in range(3))
sch = J.Schedule(Q)
fn = lambda: J.jagged_flash_attention_forward(Q, K, V, schedule=sch)  # noqa: E731
for _ in range(5):
    fn()
torch.cuda.synchronize()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    fn()
    with torch.cuda.graph(g, stream=s):
        fn()
torch.cuda.synchronize()
tg = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    tg.append(a.elapsed_time(b))
sq = float((ln.astype(np.float64) ** 2).sum())
print(f"cfg2 fwd eager {np.median(ts) * 1e3:.1f} us  graph {np.median(tg) * 1e3:.1f} us  "
      f"({4 * sq * H * D / np.median(tg) / 1e9:.1f} TF/s graph)  sum_B={S} max={ln.max()} sum_sq={int(sq)}")
