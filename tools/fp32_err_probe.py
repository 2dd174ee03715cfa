"""fp32-mode attention error vs an fp64 torch reference (diagnostic, GPU only): norm-wise and RMS-floored
elementwise relative errors of out/lse/dq/dk/dv on multi-block samples; JG_FP32_SIMT=1 selects the FFMA kernels."""
import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import restated as R
from tests.test_gpu_attention import _dense_sample_ref64
from paper_2409_15373_b200 import jagged as J
DEV = 'cuda'
for D in (64, 128):
    ln = np.array([1500, 1, 0, 129, 700, 64, 65, 1023, 257], np.int64)
    off = R.make_offsets(ln); S, H = int(off[-1]), 2
    g = torch.Generator(device=DEV).manual_seed(11)
    q, k, v, go = ((torch.rand(S, H, D, device=DEV, generator=g) * 2 - 1) for _ in range(4))
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), a, off)
    Q, K, V, G = T(q), T(k), T(v), T(go)
    saved = J.jagged_flash_attention_forward(Q, K, V); gr = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    ref = [np.zeros((S, H, D)), np.zeros((H, S)), np.zeros((S, H, D)), np.zeros((S, H, D)), np.zeros((S, H, D))]
    for i in np.nonzero(ln)[0]:
        a, b = int(off[i]), int(off[i + 1])
        outs = _dense_sample_ref64(q[a:b], k[a:b], v[a:b], go[a:b])
        ref[0][a:b], ref[1][:, a:b], ref[2][a:b], ref[3][a:b], ref[4][a:b] = (t.cpu().numpy() for t in outs)
    for got, r, nm in zip((saved.output.values, saved.logsumexp, gr.dq.values, gr.dk.values, gr.dv.values), ref, ("out","lse","dq","dk","dv")):
        gg = got.double().cpu().numpy().reshape(-1); rr = r.reshape(-1)
        rms = np.sqrt(np.mean(rr*rr)); err = np.abs(gg-rr)
        print(os.environ.get('JG_FP32_SIMT','x3'), D, nm, f"norm {np.linalg.norm(gg-rr)/np.linalg.norm(rr):.2e} max_el {np.max(err/np.maximum(np.abs(rr), rms)):.2e}")
