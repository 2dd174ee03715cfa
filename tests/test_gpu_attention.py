"""GPU parity of jagged flash attention (forward + backward) and the unfused jagged attention.

All results go through the C-ABI; the oracle (binary64, pinned to the reference) runs per head on
the same rounded inputs. fp32 mode: 1e-5 relative (norm-wise + RMS-floored elementwise). bf16:
2e-2 max-abs. Edge cases follow SPEC.md:280-300 (Bi=0 rows do not exist, Bi=1 -> out = v,
dv = grad_out, dq = dk = 0) and block-size invariance.
"""
import numpy as np
import pytest
import torch

from oracle import restated as R
from tests.parity import assert_bf16_close, assert_fp32_close, bf16_round, f32_round

pytestmark = pytest.mark.gpu
J = pytest.importorskip("paper_2409_15373_b200.jagged")
DEV = "cuda"


def make(ln, H, D, seed, dtype):
    ln = np.asarray(ln, np.int64)
    off = R.make_offsets(ln)
    S = int(off[-1])
    rnd = f32_round if dtype == torch.float32 else bf16_round
    vals = rnd(R.Rng(seed + 1).uniform_values(4 * S * H * D))
    q, k, v, go = (vals[i * S * H * D:(i + 1) * S * H * D].reshape(S, H, D) for i in range(4))
    toj = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), torch.from_numpy(a).to(dtype).to(DEV), off)  # noqa
    return off, (q, k, v, go), tuple(toj(a) for a in (q, k, v, go))


def oracle_per_head(off, q, k, v, go):
    S, H, D = q.shape
    out, lse = np.empty_like(q), np.empty((H, S))
    dq, dk, dv = np.empty_like(q), np.empty_like(q), np.empty_like(q)
    for h in range(H):
        o_h, l_h = R.jfa_forward(off, q[:, h], k[:, h], v[:, h], 64, 64)
        out[:, h], lse[h] = o_h, l_h
        dq[:, h], dk[:, h], dv[:, h] = R.jfa_backward(off, q[:, h], k[:, h], v[:, h], go[:, h], o_h, l_h, 64)
    return out, lse, dq, dk, dv


CASES = [
    ([0, 1, 2, 5, 7, 17, 33, 70, 130, 257], 1, 16),
    ([3, 0, 128, 129, 255, 1, 64], 2, 64),
    ([200, 5, 300, 0, 131], 2, 128),
    ([33, 0, 1, 190, 64, 65], 3, 32),
    (list(R.gen_lengths("zipf", 512, 0, 24, 1.1)), 1, 64),
    # forward packing (layout.cu): windows with > 32 packed samples, samples crossing 128-row windows, a sample
    # filling a window, empty samples inside a pack
    ([1] * 70 + [2, 0, 2] * 20 + [60, 3, 126, 1, 5, 128, 0, 127] + [1] * 150 + [9, 250], 2, 64),
]


@pytest.mark.parametrize("ln,H,D", CASES)
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_flash_attention_fwd_bwd(ln, H, D, mode):
    dtype = torch.float32 if mode == "fp32" else torch.bfloat16
    close = assert_fp32_close if mode == "fp32" else assert_bf16_close
    off, (q, k, v, go), (Q, K, V, G) = make(ln, H, D, 5, dtype)
    out, lse, dq, dk, dv = oracle_per_head(off, q, k, v, go)
    saved = J.jagged_flash_attention_forward(Q, K, V, 64, 64)
    close(saved.output.values, out, what="out")
    # lse is always float32; fp32-mode tolerance on it in both modes (bf16 inputs are exact in the oracle)
    assert_fp32_close(saved.logsumexp, lse, tol=1e-5 if mode == "fp32" else 2e-3, what="lse")
    # backward uses the oracle's saved state semantics: recompute from q, k, lse of the device forward
    grads = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    close(grads.dq.values, dq, what="dq")
    close(grads.dk.values, dk, what="dk")
    close(grads.dv.values, dv, what="dv")


def test_flash_attention_golden(golden):
    """The reference's own JFA outputs (tests/golden/attention.npz, binary64 inputs) in fp32 mode."""
    a = golden["attention"]
    off = a["offsets"]
    toj = lambda x: J.JaggedTensor(torch.from_numpy(off).to(DEV), torch.from_numpy(x).float().to(DEV), off)  # noqa
    Q, K, V, G = (toj(a[n]) for n in ("q", "k", "v", "go"))
    saved = J.jagged_flash_attention_forward(Q, K, V, 3, 3)
    assert_fp32_close(saved.output.values, a["out_b3x3"], tol=2e-5, what="out")
    fin = np.isfinite(a["lse_b3x3"])
    assert fin.all()  # empty segments have no rows
    assert_fp32_close(saved.logsumexp.reshape(-1), a["lse_b3x3"], tol=2e-5, what="lse")
    g = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    assert_fp32_close(g.dq.values, a["dq_b3x3"], tol=5e-5, what="dq")
    assert_fp32_close(g.dk.values, a["dk_b3x3"], tol=5e-5, what="dk")
    assert_fp32_close(g.dv.values, a["dv_b3x3"], tol=5e-5, what="dv")
    # unfused jagged attention
    assert_fp32_close(J.jagged_attention(Q, K, V).values, a["jagged_attention"], tol=2e-5, what="unfused")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_single_row_segments(dtype):
    """Bi=1 everywhere -> out = v, dv = grad_out, dq = dk = 0."""
    off, (q, k, v, go), (Q, K, V, G) = make([1] * 37, 2, 64, 9, dtype)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    torch.testing.assert_close(saved.output.values, V.values, rtol=0, atol=0)
    g = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    torch.testing.assert_close(g.dv.values.float(), G.values.float(), rtol=1e-6, atol=1e-6)
    assert float(g.dq.values.abs().max()) < 1e-5 and float(g.dk.values.abs().max()) < 1e-5


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_uniform_keys_average_values(dtype):
    """all keys equal within a segment -> every output row = mean of the segment's V."""
    ln = [5, 140, 3]
    off, (q, k, v, go), (Q, K, V, G) = make(ln, 1, 64, 2, dtype)
    kk = np.repeat(k[off[:-1]][:, None], 1, 1)
    kconst = np.concatenate([np.repeat(k[off[i]:off[i] + 1], ln[i], 0) for i in range(3)])
    Kc = J.JaggedTensor(K.offsets, torch.from_numpy(kconst).to(dtype).to(DEV), off)
    out = J.jagged_flash_attention_forward(Q, Kc, V).output.values.double().cpu().numpy()
    for i in range(3):
        seg = slice(off[i], off[i + 1])
        np.testing.assert_allclose(out[seg], np.broadcast_to(v[seg].mean(0), out[seg].shape),
                                   atol=2e-2 if dtype == torch.bfloat16 else 1e-5)
    del kk


def test_zero_grad_out_gives_zero_grads():
    off, _, (Q, K, V, G) = make([7, 0, 150], 1, 64, 3, torch.bfloat16)
    Z = J.JaggedTensor(G.offsets, torch.zeros_like(G.values), off)
    g = J.jagged_flash_attention_backward(Q, K, V, Z, J.jagged_flash_attention_forward(Q, K, V))
    for t in (g.dq, g.dk, g.dv):
        assert float(t.values.abs().max()) == 0.0


def test_block_size_invariance_and_errors():
    off, _, (Q, K, V, G) = make([9, 33], 1, 16, 4, torch.float32)
    a = J.jagged_flash_attention_forward(Q, K, V, 1, 1).output.values
    b = J.jagged_flash_attention_forward(Q, K, V, 64, 64).output.values
    assert torch.equal(a, b)
    with pytest.raises(J.JaggedError, match="block sizes must be >= 1"):
        J.jagged_flash_attention_forward(Q, K, V, 0, 64)
    K2 = J.JaggedTensor(torch.from_numpy(R.make_offsets([10, 32])).to(DEV), K.values, R.make_offsets([10, 32]))
    with pytest.raises(J.JaggedError, match="q, k, v must share offsets"):
        J.jagged_flash_attention_forward(Q, K2, V)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    saved.logsumexp = saved.logsumexp[:, :5]
    with pytest.raises(J.JaggedError, match="saved state does not match inputs"):
        J.jagged_flash_attention_backward(Q, K, V, G, saved)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_unfused_matches_flash(dtype):
    off, (q, k, v, go), (Q, K, V, G) = make([4, 0, 33, 70], 2, 32, 6, dtype)
    ref = np.stack([R.jagged_attention(off, q[:, h], k[:, h], v[:, h]) for h in range(2)], 1)
    got = J.jagged_attention(Q, K, V).values
    if dtype == torch.float32:
        assert_fp32_close(got, ref, what="unfused")
    else:
        assert_bf16_close(got, ref, tol=3e-2, what="unfused (bf16 scores materialized)")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_fwd_bwd_host_entry_matches_device_api(dtype):
    """jg_jagged_flash_attention_fwd_bwd_host (pinned host buffers, chunked three-stream copy/compute pipeline)
    gives the device API's results on every sample (the path bench.py's e2e measures); fp32 runs the tcgen05
    fp16 two-piece kernels on concurrent streams."""
    from paper_2409_15373_b200 import _lib
    ln = list(R.gen_lengths("half-mean", 300, 4, 40))
    H, D = 2, 128
    off, (q, k, v, go), (Q, K, V, G) = make(ln, H, D, 9, dtype)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    grads = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    S = int(off[-1])
    host = [torch.from_numpy(a).to(dtype).pin_memory() for a in (q, k, v, go)]
    outs = [torch.empty(S, H, D, dtype=dtype).pin_memory() for _ in range(4)]
    lse = torch.empty(H, S, dtype=torch.float32).pin_memory()
    hoff = np.ascontiguousarray(off, np.int64)
    _lib.check(_lib.lib().jg_jagged_flash_attention_fwd_bwd_host(
        hoff.ctypes.data, len(ln), H, D, *(t.data_ptr() for t in host), outs[0].data_ptr(), lse.data_ptr(),
        outs[1].data_ptr(), outs[2].data_ptr(), outs[3].data_ptr(), 1 if dtype == torch.bfloat16 else 0, None))
    close = assert_bf16_close if dtype == torch.bfloat16 else assert_fp32_close
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
    close(outs[0], saved.output.values.double().cpu().numpy(), tol=tol, what="out")
    np.testing.assert_allclose(lse.numpy(), saved.logsumexp.cpu().numpy(), rtol=1e-5, atol=1e-4)
    for got, ref, name in zip(outs[1:], (grads.dq, grads.dk, grads.dv), ("dq", "dk", "dv")):
        close(got, ref.values.double().cpu().numpy(), tol=tol, what=name)


def test_unfused_tensor_core_path_multihead():
    """jagged_attention on the tcgen05 grouped GEMM (bf16, head_dim 128, two heads: TMA head coordinate, strided
    output) and on a jagged^2 scratch whose size is not a multiple of 16 bytes."""
    off, (q, k, v, go), (Q, K, V, G) = make([3, 129, 0, 70, 255], 2, 128, 8, torch.bfloat16)
    ref = np.stack([R.jagged_attention(off, q[:, h], k[:, h], v[:, h]) for h in range(2)], 1)
    assert_bf16_close(J.jagged_attention(Q, K, V).values, ref, tol=3e-2, what="unfused tcgen05 (2 heads)")


def _dense_sample_ref(q, k, v, go):
    """fp32 torch reference of one sample's attention fwd + bwd ([n, H, D] inputs)."""
    D = q.shape[-1]
    q, k, v, go = (t.float().transpose(0, 1).requires_grad_() for t in (q, k, v, go))  # [H, n, D]
    s = torch.matmul(q, k.transpose(1, 2)) / D ** 0.5
    lse = torch.logsumexp(s, dim=-1)
    o = torch.matmul(torch.softmax(s, dim=-1), v)
    dq, dk, dv = torch.autograd.grad(o, (q, k, v), go)
    return (o.detach().transpose(0, 1), lse.detach(), dq.transpose(0, 1), dk.transpose(0, 1), dv.transpose(0, 1))


def test_full_size_cfg3_properties():
    """BASELINE cfg3 at full size (B=1024, L=1024, D=128, H=4, half-mean seed 0): spot-check whole samples
    against an fp32 torch reference (largest, smallest non-empty, and random ones) and check the size-independent
    identities on every sample: sum_k dV_k = sum_q dO_q (rows of P sum to 1; relative to sum_q |dO_q|) and
    sum_k dK_k = 0 (rows of dS sum to 0; max-abs). bf16 tolerance 2e-2."""
    ln = R.gen_lengths("half-mean", 1024, 0, 1024)
    off = R.make_offsets(ln)
    S, H, D = int(off[-1]), 4, 128
    g = torch.Generator(device=DEV).manual_seed(3)
    q, k, v, go = ((torch.rand(S, H, D, device=DEV, generator=g) * 2 - 1).bfloat16() for _ in range(4))
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), a, off)  # noqa: E731
    Q, K, V, G = T(q), T(k), T(v), T(go)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    gr = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    nz = np.nonzero(ln)[0]
    picks = {int(nz[np.argmax(ln[nz])]), int(nz[np.argmin(ln[nz])])} | set(np.random.default_rng(0).choice(nz, 4).tolist())
    for i in sorted(picks):
        a, b = int(off[i]), int(off[i + 1])
        o, lse, dq, dk, dv = _dense_sample_ref(q[a:b], k[a:b], v[a:b], go[a:b])
        assert_bf16_close(saved.output.values[a:b], o.cpu().numpy(), what=f"out sample {i} (n={b - a})")
        assert_bf16_close(saved.logsumexp[:, a:b], lse.cpu().numpy(), what=f"lse sample {i}")
        for got, ref, nm in ((gr.dq, dq, "dq"), (gr.dk, dk, "dk"), (gr.dv, dv, "dv")):
            assert_bf16_close(got.values[a:b], ref.cpu().numpy(), what=f"{nm} sample {i} (n={b - a})")
    seg = torch.repeat_interleave(torch.arange(len(ln), device=DEV), torch.from_numpy(ln).to(DEV))
    segsum = lambda t: torch.zeros(len(ln), H, D, device=DEV).index_add_(0, seg, t.float())  # noqa: E731
    sdv, sdo, sdk = segsum(gr.dv.values), segsum(go), segsum(gr.dk.values)
    scale = segsum(go.abs()).clamp_min(1.0)
    assert float(((sdv - sdo).abs() / scale).max()) < 2e-2, "sum_k dV != sum_q dO"
    # dS is rounded to bf16 before the dK MMA, so its rows sum to 0 only up to bf16 rounding: the identity is
    # checked at the product's max-abs tolerance (sum_k |dK_k| is O(1-5) per (sample, head, d) here)
    assert float(sdk.abs().max()) < 2e-2, "sum_k dK != 0"


def _dense_sample_ref64(q, k, v, go):
    """fp64 torch reference of one sample's attention fwd + bwd ([n, H, D] inputs)."""
    D = q.shape[-1]
    q, k, v, go = (t.double().transpose(0, 1).requires_grad_() for t in (q, k, v, go))  # [H, n, D]
    s = torch.matmul(q, k.transpose(1, 2)) / D ** 0.5
    lse = torch.logsumexp(s, dim=-1)
    o = torch.matmul(torch.softmax(s, dim=-1), v)
    dq, dk, dv = torch.autograd.grad(o, (q, k, v), go)
    return (o.detach().transpose(0, 1), lse.detach(), dq.transpose(0, 1), dk.transpose(0, 1), dv.transpose(0, 1))


@pytest.mark.parametrize("D", [64, 128])
def test_fp32_tensor_core_path_multi_block(D):
    """fp32 mode on tcgen05 (attn_x3_sm100.cu, split-bf16 emulation) at sizes with many 64-key blocks and 128-row
    tiles per sample (up to 1,500 rows): every sample against an fp64 torch reference at the fp32 tolerance, and
    the results bit-identical across two runs (two deterministic passes, no atomics)."""
    ln = np.array([1500, 1, 0, 129, 700, 64, 65, 1023, 257], np.int64)
    off = R.make_offsets(ln)
    S, H = int(off[-1]), 2
    g = torch.Generator(device=DEV).manual_seed(11)
    q, k, v, go = ((torch.rand(S, H, D, device=DEV, generator=g) * 2 - 1) for _ in range(4))
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), a, off)  # noqa: E731
    Q, K, V, G = T(q), T(k), T(v), T(go)
    runs = []
    for _ in range(2):
        saved = J.jagged_flash_attention_forward(Q, K, V)
        gr = J.jagged_flash_attention_backward(Q, K, V, G, saved)
        torch.cuda.synchronize()
        runs.append((saved.output.values.clone(), saved.logsumexp.clone(), gr.dq.values.clone(),
                     gr.dk.values.clone(), gr.dv.values.clone()))
    for a, b in zip(*runs):
        assert torch.equal(a, b), "fp32 attention is not bit-identical across runs"
    out, lse, dq, dk, dv = runs[0]
    ref = [np.zeros((S, H, D)), np.zeros((H, S)), np.zeros((S, H, D)), np.zeros((S, H, D)), np.zeros((S, H, D))]
    for i in np.nonzero(ln)[0]:
        a, b = int(off[i]), int(off[i + 1])
        o, l, rq, rk, rv = _dense_sample_ref64(q[a:b], k[a:b], v[a:b], go[a:b])
        ref[0][a:b], ref[1][:, a:b], ref[2][a:b], ref[3][a:b], ref[4][a:b] = (
            t.cpu().numpy() for t in (o, l, rq, rk, rv))
    for got, r, nm in zip((out, lse, dq, dk, dv), ref, ("out", "lse", "dq", "dk", "dv")):
        assert_fp32_close(got, r, what=f"fp32 tcgen05 {nm} (D={D})")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_unaligned_views_take_scalar_kernels(dtype):
    """Tensors whose base is not 16-byte aligned (views one element into a larger buffer) must not reach the
    16-byte vector paths (TMA boxes, float4 loads): the C-ABI routes them to the row-per-warp kernels. Results agree
    with the aligned run (fp32 1e-5 / bf16 2e-2) instead of faulting."""
    ln = [5, 0, 130, 64, 257]
    off, _, (Q, K, V, G) = make(ln, 2, 64, 13, dtype)
    close = assert_fp32_close if dtype == torch.float32 else assert_bf16_close

    def shifted(t):
        buf = torch.empty(t.values.numel() + 1, dtype=dtype, device=DEV)
        view = buf[1:].view_as(t.values)
        view.copy_(t.values)
        assert view.data_ptr() % 16 != 0
        return J.JaggedTensor(t.offsets, view, off)

    Qs, Ks, Vs, Gs = (shifted(t) for t in (Q, K, V, G))
    ref = J.jagged_flash_attention_forward(Q, K, V)
    got = J.jagged_flash_attention_forward(Qs, Ks, Vs)
    close(got.output.values, ref.output.values.double().cpu().numpy(), what="out (unaligned)")
    gr = J.jagged_flash_attention_backward(Q, K, V, G, ref)
    gg = J.jagged_flash_attention_backward(Qs, Ks, Vs, Gs, got)
    for a, b, nm in ((gg.dq, gr.dq, "dq"), (gg.dk, gr.dk, "dk"), (gg.dv, gr.dv, "dv")):
        close(a.values, b.values.double().cpu().numpy(), what=f"{nm} (unaligned)")


def test_full_size_cfg3_fp32_tensor_core_path():
    """BASELINE cfg3 at full size in fp32 mode (the split-bf16 tcgen05 kernels): whole samples (largest, smallest
    non-empty, random ones) against an fp64 torch reference at the fp32 tolerance, and the size-independent
    identities on every sample: sum_k dV_k = sum_q dO_q and sum_k dK_k = 0 (to fp32 accumulation error)."""
    ln = R.gen_lengths("half-mean", 1024, 0, 1024)
    off = R.make_offsets(ln)
    S, H, D = int(off[-1]), 4, 128
    g = torch.Generator(device=DEV).manual_seed(5)
    q, k, v, go = ((torch.rand(S, H, D, device=DEV, generator=g) * 2 - 1) for _ in range(4))
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), a, off)  # noqa: E731
    Q, K, V, G = T(q), T(k), T(v), T(go)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    gr = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    nz = np.nonzero(ln)[0]
    picks = {int(nz[np.argmax(ln[nz])]), int(nz[np.argmin(ln[nz])])} | set(np.random.default_rng(1).choice(nz, 3).tolist())
    for i in sorted(picks):
        a, b = int(off[i]), int(off[i + 1])
        o, lse, dq, dk, dv = _dense_sample_ref64(q[a:b], k[a:b], v[a:b], go[a:b])
        assert_fp32_close(saved.output.values[a:b], o.cpu().numpy(), what=f"out sample {i} (n={b - a})")
        assert_fp32_close(saved.logsumexp[:, a:b], lse.cpu().numpy(), what=f"lse sample {i}")
        for got, ref, nm in ((gr.dq, dq, "dq"), (gr.dk, dk, "dk"), (gr.dv, dv, "dv")):
            assert_fp32_close(got.values[a:b], ref.cpu().numpy(), what=f"{nm} sample {i} (n={b - a})")
    seg = torch.repeat_interleave(torch.arange(len(ln), device=DEV), torch.from_numpy(ln).to(DEV))
    segsum = lambda t: torch.zeros(len(ln), H, D, device=DEV, dtype=torch.float64).index_add_(0, seg, t.double())  # noqa
    sdv, sdo, sdk = segsum(gr.dv.values), segsum(go), segsum(gr.dk.values)
    scale = segsum(go.abs()).clamp_min(1.0)
    assert float(((sdv - sdo).abs() / scale).max()) < 1e-5, "sum_k dV != sum_q dO"
    assert float((sdk.abs() / segsum(gr.dk.values.abs()).clamp_min(1.0)).max()) < 1e-5, "sum_k dK != 0"


@pytest.mark.parametrize("scales", [(1e3, 1e-3, 1e2, 1e-2), (1e-3, 1e3, 1e-4, 1e4), (3e-2, 30.0, 5e3, 2e-3)])
def test_fp32_tensor_core_path_operand_magnitudes(scales):
    """The fp16 two-piece path rescales every operand by a power of two before splitting (fp16 covers ~6e-5 .. 65504):
    q, k, v, dO of very different magnitudes must still match an fp64 torch reference at the fp32 tolerance."""
    sq, sk, sv, sg = scales
    ln = np.array([300, 1, 129, 0, 64], np.int64)
    off = R.make_offsets(ln)
    S, H, D = int(off[-1]), 2, 128
    g = torch.Generator(device=DEV).manual_seed(17)
    q, k, v, go = ((torch.rand(S, H, D, device=DEV, generator=g) * 2 - 1) * s for s in (sq, sk, sv, sg))
    # sq * sk = 1 keeps the scores q.k / sqrt(D) O(1): a saturated softmax would make dq / dk vanish (ill-conditioned)
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), a, off)  # noqa: E731
    Q, K, V, G = T(q), T(k), T(v), T(go)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    gr = J.jagged_flash_attention_backward(Q, K, V, G, saved)
    for i in np.nonzero(ln)[0]:
        a, b = int(off[i]), int(off[i + 1])
        o, lse, dq, dk, dv = _dense_sample_ref64(q[a:b], k[a:b], v[a:b], go[a:b])
        assert_fp32_close(saved.output.values[a:b], o.cpu().numpy(), what=f"out sample {i} scales {scales}")
        assert_fp32_close(saved.logsumexp[:, a:b], lse.cpu().numpy(), what=f"lse sample {i}")
        for got, ref, nm in ((gr.dq, dq, "dq"), (gr.dk, dk, "dk"), (gr.dv, dv, "dv")):
            if b - a == 1 and nm != "dv":  # a one-row sample's dq / dk are exactly 0 in the reference
                continue
            assert_fp32_close(got.values[a:b], ref.cpu().numpy(), what=f"{nm} sample {i} scales {scales}")
