"""GPU parity of the padded dense_flash_attention mode (attention.cpp:106-160) through the C-ABI.

The same tcgen05 / SIMT kernels run with segments of max_len rows (offsets i*L) and per-sample valid lengths:
keys past a length are masked, rows past it are zero with lse = -inf. Checked against the binary64 oracle
(pinned to the compiled reference by tests/test_oracle.py::test_dense_flash_*), and — at larger sizes —
against the jagged mode on the compacted rows (masked keys contribute exact zeros, so the valid rows match).
fp32 mode: 1e-5 relative; bf16: 2e-2 max-abs.
"""
import numpy as np
import pytest
import torch

from oracle import restated as R
from tests.parity import assert_bf16_close, assert_fp32_close, bf16_round, f32_round

pytestmark = pytest.mark.gpu
J = pytest.importorskip("paper_2409_15373_b200.jagged")
DEV = "cuda"


def padded_inputs(ln, L, H, D, seed, dtype):
    rnd = f32_round if dtype == torch.float32 else bf16_round
    B = len(ln)
    vals = rnd(R.Rng(seed).uniform_values(4 * B * L * H * D))  # padding rows hold finite values too
    return [vals[i * B * L * H * D:(i + 1) * B * L * H * D].reshape(B, L, H, D) for i in range(4)]


def oracle(ln, q, k, v, go):
    """Per head: dense_flash_attention (out, lse) and the gradients of the valid rows (jagged oracle on the
    compacted rows), zero past each length."""
    B, L, H, D = q.shape
    out, lse = np.zeros_like(q), np.full((H, B * L), -np.inf)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    off = R.make_offsets(ln)
    rows = np.concatenate([i * L + np.arange(n) for i, n in enumerate(ln)]).astype(np.int64) if len(ln) else []
    for h in range(H):
        o_h, l_h = R.dense_flash_attention(ln, q[:, :, h], k[:, :, h], v[:, :, h], 64, 64)
        out[:, :, h], lse[h] = o_h, l_h
        cq, ck, cv, cg = (a[:, :, h].reshape(B * L, D)[rows] for a in (q, k, v, go))
        co, cl = R.jfa_forward(off, cq, ck, cv, 64, 64)
        g = R.jfa_backward(off, cq, ck, cv, cg, co, cl, 64)
        for dst, src in zip((dq, dk, dv), g):
            flat = dst[:, :, h].reshape(B * L, D)
            flat[rows] = src
            dst[:, :, h] = flat.reshape(B, L, D)
    return out, lse, dq, dk, dv


CASES = [([5, 0, 9, 3], 9, 1, 16), ([0, 1, 130, 257, 200, 64], 257, 2, 64), ([128, 3, 255, 0, 256], 256, 2, 128),
         ([300, 17, 1, 299], 300, 1, 128)]


@pytest.mark.parametrize("ln,L,H,D", CASES)
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_dense_flash_fwd_bwd(ln, L, H, D, mode):
    dtype = torch.float32 if mode == "fp32" else torch.bfloat16
    close = assert_fp32_close if mode == "fp32" else assert_bf16_close
    q, k, v, go = padded_inputs(ln, L, H, D, 7, dtype)
    out, lse, dq, dk, dv = oracle(np.asarray(ln, np.int64), q, k, v, go)
    T = lambda a: torch.from_numpy(a).to(dtype).to(DEV)  # noqa: E731
    Q, K, V, G = T(q), T(k), T(v), T(go)
    saved = J.dense_flash_attention(Q, K, V, ln)
    # compare the valid rows (the RMS floor of the fp32 tolerance is taken over them) and require exact
    # zeros past each length
    B = len(ln)
    vm = (np.arange(L)[None, :] < np.asarray(ln)[:, None]).reshape(-1)
    vt = torch.from_numpy(vm).to(DEV)

    def close_rows(got, ref, what):
        g = got.reshape(B * L, H, D)
        close(g[vt], ref.reshape(B * L, H, D)[vm], what=what)
        assert not g[~vt].any(), f"{what}: rows past each length must be zero"

    close_rows(saved.output, out, "out")
    got_lse = saved.logsumexp.cpu().numpy()
    assert np.array_equal(np.isinf(got_lse), np.isinf(lse)), "lse -inf pattern (rows past each length)"
    fin = np.isfinite(lse)
    assert_fp32_close(saved.logsumexp[torch.from_numpy(fin).to(DEV)], lse[fin],
                      tol=1e-5 if mode == "fp32" else 2e-3, what="lse")
    gq, gk, gv = J.dense_flash_attention_backward(Q, K, V, G, saved, ln)
    close_rows(gq, dq, "dq")
    close_rows(gk, dk, "dk")
    close_rows(gv, dv, "dv")


def test_dense_flash_single_head_layout_and_reference_shape():
    """[B, L, D] inputs (the reference's DenseTensor shape) behave as one head."""
    ln, L, D = [4, 7, 0], 7, 32
    q, k, v, _ = (a[:, :, 0] for a in padded_inputs(ln, L, 1, D, 3, torch.float32))
    saved = J.dense_flash_attention(*(torch.from_numpy(a).float().to(DEV) for a in (q, k, v)), np.asarray(ln), 3, 5)
    o, l_ = R.dense_flash_attention(ln, q, k, v, 3, 5)
    assert saved.output.shape == (3, L, D)
    assert_fp32_close(saved.output, o, what="out")
    assert not saved.output[2].any() and torch.isinf(saved.logsumexp[0, 2 * L:]).all()


@pytest.mark.parametrize("D", [64, 128])
def test_dense_flash_valid_rows_match_jagged_mode(D):
    """Full-size property (cfg3-like lengths): padded-mode rows inside each length equal the jagged kernels on
    the compacted tensors; rows past the length are exactly zero."""
    B, L, H = 64, 1024, 2
    ln = R.gen_lengths("half-mean", L, 0, B)
    off = R.make_offsets(ln)
    g = torch.Generator(device=DEV).manual_seed(0)
    q, k, v, go = ((torch.rand(B, L, H, D, device=DEV, generator=g) * 2 - 1).bfloat16() for _ in range(4))
    lens = torch.from_numpy(ln).to(DEV)
    valid = (torch.arange(L, device=DEV)[None, :] < lens[:, None]).reshape(-1)
    comp = lambda a: J.JaggedTensor(torch.from_numpy(off).to(DEV), a.reshape(B * L, H, D)[valid].contiguous(), off)  # noqa
    saved = J.dense_flash_attention(q, k, v, ln)
    js = J.jagged_flash_attention_forward(comp(q), comp(k), comp(v))
    po = saved.output.reshape(B * L, H, D)
    assert_bf16_close(po[valid], js.output.values.float().cpu().numpy(), what="valid rows vs jagged")
    assert not po[~valid].any(), "rows past each length must be zero"
    if D == 128:
        gq, gk, gv = J.dense_flash_attention_backward(q, k, v, go, saved, ln)
        jg = J.jagged_flash_attention_backward(comp(q), comp(k), comp(v), comp(go), js)
        for a, b, nm in ((gq, jg.dq, "dq"), (gk, jg.dk, "dk"), (gv, jg.dv, "dv")):
            a = a.reshape(B * L, H, D)
            assert_bf16_close(a[valid], b.values.float().cpu().numpy(), what=nm)
            assert not a[~valid].any(), f"{nm} rows past each length must be zero"


def test_dense_flash_errors():
    x = torch.zeros(2, 4, 8, device=DEV)
    with pytest.raises(J.JaggedError, match=r"dense_flash_attention: sample 1 length 5 out of bounds for L=4"):
        J.dense_flash_attention(x, x, x, [1, 5])
    with pytest.raises(J.JaggedError, match="dense_flash_attention: lengths size mismatch"):
        J.dense_flash_attention(x, x, x, [1])
    with pytest.raises(J.JaggedError, match=r"dense_flash_attention: q, k, v must share a \[B, L, D\] shape"):
        J.dense_flash_attention(x, torch.zeros(2, 4, 4, device=DEV), x, [1, 2])
    with pytest.raises(J.JaggedError, match="dense_flash_attention: block sizes must be >= 1"):
        J.dense_flash_attention(x, x, x, [1, 2], 0, 4)
