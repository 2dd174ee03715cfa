"""Host-side cost of one JFA forward call (diagnostic, GPU only): enqueue time per call of the Python API, the raw
C-ABI call with preallocated outputs, and the pieces of the Python wrapper. cfg2 workload."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2409_15373_b200 import jagged as J, synth, _lib  # noqa: E402

ln = synth.gen_lengths("zipf", 512, 0, 256, 1.1)
off = synth.offsets_of(ln)
S, D, H = int(off[-1]), 64, 1
mk = lambda: (torch.rand(S, H, D, device='cuda') * 2 - 1).bfloat16()  # noqa: E731
Q, K, V = (J.JaggedTensor(torch.from_numpy(off).cuda(), mk(), off) for _ in range(3))
sch = J.Schedule(Q)
out = torch.empty_like(Q.values)
lse = torch.empty(H, S, dtype=torch.float32, device='cuda')
lib = _lib.lib()


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    return dt * 1e6


st = torch.cuda.current_stream().cuda_stream
print(f"python API forward        {per_call(lambda: J.jagged_flash_attention_forward(Q, K, V, schedule=sch)):7.2f} us/call")
raw = lambda: lib.jg_jagged_flash_attention_forward(Q.offsets.data_ptr(), Q.batch, Q.total_rows, H, D,  # noqa: E731
                                                    Q.values.data_ptr(), K.values.data_ptr(), V.values.data_ptr(), 64,
                                                    64, out.data_ptr(), lse.data_ptr(), J._dt(Q.values), sch.handle, st)
print(f"raw C-ABI forward         {per_call(raw):7.2f} us/call")
print(f"validation                {per_call(lambda: J._require_attention_inputs(Q, K, V, 'x')):7.2f} us/call")
print(f"torch.empty_like x2       {per_call(lambda: (torch.empty_like(Q.values), torch.empty(H, S, dtype=torch.float32, device='cuda'))):7.2f} us/call")
print(f"with_values               {per_call(lambda: Q.with_values(out)):7.2f} us/call")
print(f"current_stream            {per_call(lambda: torch.cuda.current_stream().cuda_stream):7.2f} us/call")
