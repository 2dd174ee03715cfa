"""GPU parity of the jagged softmax kernels across their internal paths (linalg.cpp:98-120, :199-220, :355-388,
:474-507) against the oracle (oracle/jagged_oracle.c, pinned by tests/test_oracle.py).

jagged2_softmax keeps a row in registers as the aligned 16-byte chunks that overlap it (rows up to 1273 bf16 /
637 fp32 elements), writes the wholly covered chunks with one store and the two edge chunks element-wise, and
takes a two-pass loop for longer rows; the lengths below put rows at every element alignment, on both sides of
the register cap, and next to one another (edge chunks shared between rows written by different warps).
jagged_softmax is checked on segments both sides of its shared-memory slab cap. fp32 mode within 1e-5
(norm-wise relative), bf16 within 2e-2 max-abs (|p| <= 1).
"""
import numpy as np
import pytest
import torch

from oracle import restated as R
from tests.parity import assert_bf16_close, assert_fp32_close

pytestmark = pytest.mark.gpu

J = pytest.importorskip("paper_2409_15373_b200.jagged")

DEV = "cuda"
J2_LENGTHS = [1, 3, 0, 7, 9, 636, 637, 638, 5, 1273, 1274, 1500, 2, 31, 33, 100]
JS_LENGTHS = [0, 1, 5, 95, 96, 97, 767, 768, 769, 1024, 1600, 3]


def _assert_softmax_vjp_fp32(got, ref, off, p, g, tol=1e-5):
    """fp32 VJP: norm-wise 1e-5, and elementwise against the conditioning of ds_i = p_i (g_i - dot): an fp32
    evaluation perturbs dot by ~u sum_j |g_j| p_j, which ds_i inherits times p_i (cancellation in g_i - dot), so
    |err_i| <= tol (|ds_i| + p_i (|g_i| + sum_j |g_j p_j|)) per row."""
    g64 = np.asarray(got.double().cpu().numpy(), np.float64).reshape(-1)
    err = np.abs(g64 - ref)
    assert float(np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-300)) <= tol
    sqo = R.sq_offsets(off)
    for i in range(len(off) - 1):
        n = int(off[i + 1] - off[i])
        if n == 0:
            continue
        sl = slice(int(sqo[i]), int(sqo[i]) + n * n)
        pb, gb = p[sl].reshape(n, n), g[sl].reshape(n, n)
        scale = np.abs(gb * pb).sum(axis=1, keepdims=True)
        bound = tol * (np.abs(ref[sl].reshape(n, n)) + pb * (np.abs(gb) + scale)) + 1e-30
        bad = np.argwhere(err[sl].reshape(n, n) > bound)
        assert bad.size == 0, f"jagged2 vjp sample {i}: {len(bad)} elements out of bound, first {bad[0]}"


def _close(mode):
    return assert_fp32_close if mode == "fp32" else assert_bf16_close


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_jagged2_softmax_paths(mode):
    ln = np.asarray(J2_LENGTHS, np.int64)
    off = R.make_offsets(ln)
    sq = int((ln * ln).sum())
    dt = torch.float32 if mode == "fp32" else torch.bfloat16
    a = (R.Rng(5).uniform_values(sq) * 6.0).astype(np.float64)
    go = R.Rng(6).uniform_values(sq)
    at, gt = torch.from_numpy(a).to(dt), torch.from_numpy(go).to(dt)
    a_in, g_in = at.double().numpy(), gt.double().numpy()  # the oracle sees the rounded inputs
    offd = torch.from_numpy(off).to(DEV)
    A = J.Jagged2Tensor(offd, at.to(DEV), off)
    G = J.Jagged2Tensor(offd, gt.to(DEV), off)
    _close(mode)(J.jagged2_softmax(A).values, R.jagged2_softmax(off, a_in), what="jagged2_softmax")
    got = J.jagged2_softmax_vjp(A, G).values
    ref = R.jagged2_softmax_vjp(off, a_in, g_in)
    if mode == "bf16":
        assert_bf16_close(got, ref, what="jagged2 vjp")
    else:
        _assert_softmax_vjp_fp32(got, ref, off, R.jagged2_softmax(off, a_in), g_in)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_jagged2_softmax_neighbour_rows_untouched(mode):
    """Edge chunks are shared with the neighbouring rows: a sentinel-filled output must only change inside rows."""
    ln = np.asarray([3, 5, 2, 7, 1, 9], np.int64)
    off = R.make_offsets(ln)
    sq = int((ln * ln).sum())
    dt = torch.float32 if mode == "fp32" else torch.bfloat16
    a = torch.from_numpy(R.Rng(9).uniform_values(sq)).to(dt)
    A = J.Jagged2Tensor(torch.from_numpy(off).to(DEV), a.to(DEV), off)
    p = J.jagged2_softmax(A).values.double().cpu().numpy()
    ref = R.jagged2_softmax(off, a.double().numpy())
    _close(mode)(torch.from_numpy(p), ref, what="jagged2_softmax small rows")
    # every row sums to one
    for i, n in enumerate(ln):
        blk = p[R.sq_offsets(off)[i]:R.sq_offsets(off)[i] + n * n].reshape(n, n)
        np.testing.assert_allclose(blk.sum(axis=1), 1.0, atol=2e-2 if mode == "bf16" else 1e-6)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
@pytest.mark.parametrize("D", [8, 64, 256, 200])
def test_jagged_softmax_paths(mode, D):
    ln = np.asarray(JS_LENGTHS, np.int64)
    off = R.make_offsets(ln)
    S = int(ln.sum())
    dt = torch.float32 if mode == "fp32" else torch.bfloat16
    x = torch.from_numpy((R.Rng(7).uniform_values(S * D) * 6.0).reshape(S, D)).to(dt)
    g = torch.from_numpy(R.Rng(8).uniform_values(S * D).reshape(S, D)).to(dt)
    offd = torch.from_numpy(off).to(DEV)
    X = J.JaggedTensor(offd, x.to(DEV), off)
    G = J.JaggedTensor(offd, g.to(DEV), off)
    xi, gi = x.double().numpy(), g.double().numpy()
    p = R.jagged_softmax(off, xi)
    _close(mode)(J.jagged_softmax(X).values, p, what="jagged_softmax")
    got, ref = J.jagged_softmax_vjp(X, G).values, R.jagged_softmax_vjp(off, xi, gi)
    if mode == "bf16":
        assert_bf16_close(got, ref, what="jagged_softmax vjp")
        return
    # fp32: the conditioned bound of _assert_softmax_vjp_fp32, per (segment, column)
    g64 = got.double().cpu().numpy()
    err = np.abs(g64 - ref)
    assert float(np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-300)) <= 1e-5
    for i in range(len(ln)):
        sl = slice(int(off[i]), int(off[i + 1]))
        scale = np.abs(gi[sl] * p[sl]).sum(axis=0, keepdims=True)
        bound = 1e-5 * (np.abs(ref[sl]) + p[sl] * (np.abs(gi[sl]) + scale)) + 1e-30
        assert not (err[sl] > bound).any(), f"jagged_softmax vjp segment {i}"
