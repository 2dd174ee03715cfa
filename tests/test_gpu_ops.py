"""GPU parity of the offsets layer, layout conversions and the Table-1 operators + VJPs.

Every device result goes through the C-ABI (libjagged_b200.so) and is compared with the oracle
(oracle/jagged_oracle.c, pinned to the reference by tests/test_oracle.py) on identical inputs:
integer/layout work bit-exact; fp32 mode within 1e-5 relative; bf16 inputs within 2e-2 max-abs
(fp32 outputs, since bf16 cannot hold |x|~30 outputs to 2e-2 — SURVEY.md §7).
"""
import numpy as np
import pytest
import torch

from oracle import restated as R
from tests.parity import assert_bf16_close, assert_fp32_close, bf16_round, f32_round

pytestmark = pytest.mark.gpu

J = pytest.importorskip("paper_2409_15373_b200.jagged")

DEV = "cuda"


def jt(off, vals, dtype=torch.float32):
    return J.JaggedTensor(torch.from_numpy(np.asarray(off, np.int64)).to(DEV),
                          torch.from_numpy(np.asarray(vals)).to(dtype).to(DEV), np.asarray(off, np.int64))


def rand(n, seed):
    return R.Rng(seed).uniform_values(n)


LENGTH_SETS = {
    "golden": [0, 1, 2, 5, 7, 17, 33, 70],
    "uniform": list(R.gen_lengths("uniform", 128, 0, 64)),       # BASELINE cfg1 lengths
    "long": [0, 130, 1, 257, 64, 128, 0],
}


# ------------------------------------------------------------------ offsets layer / scheduler
def test_offsets_layer_bit_exact():
    for name, ln in LENGTH_SETS.items():
        ln = np.asarray(ln, np.int64)
        x = J.make_jagged(ln, torch.zeros(int(ln.sum()), 3, device=DEV))
        np.testing.assert_array_equal(x.offsets.cpu().numpy(), R.make_offsets(ln), err_msg=name)
        s2 = J.Jagged2Tensor(x.offsets, torch.zeros(int((ln * ln).sum()), device=DEV), x.host_offsets)
        np.testing.assert_array_equal(s2.sq_offsets.cpu().numpy(), R.sq_offsets(R.make_offsets(ln)))
    big = R.gen_lengths("half-mean", 1024, 0, 1024)
    x = J.make_jagged(big, torch.zeros(int(big.sum()), 1, device=DEV))
    np.testing.assert_array_equal(x.offsets.cpu().numpy(), R.make_offsets(big))
    with pytest.raises(J.JaggedError, match="make_jagged: negative length at sample 2"):
        J.make_jagged([1, 2, -1], torch.zeros(3, 1, device=DEV))


def expected_work_list(ln, tile=128, max_bins=64):
    items = []
    nb = [(int(n) + tile - 1) // tile for n in ln]
    for b in range(max_bins, 0, -1):
        for i, n in enumerate(nb):
            if n > 0 and min(n, max_bins) == b:
                items += [(i, t) for t in range(n)]
    return np.asarray(items, np.int32).reshape(-1, 2)


@pytest.mark.parametrize("lens", [
    R.gen_lengths("half-mean", 1024, 0, 1024),
    R.gen_lengths("zipf", 512, 0, 256, 1.1),
    np.array([0, 0, 5, 9000, 300, 128, 129, 0]),
])
def test_lpt_work_list(lens):
    x = jt(R.make_offsets(lens), np.zeros((int(np.sum(lens)), 1), np.float32))
    got = J.Schedule(x).work_list()
    np.testing.assert_array_equal(got, expected_work_list(lens))


# ------------------------------------------------------------------ layout conversions (bit-exact)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_layout_conversions_bit_exact(dtype):
    ln = np.array([0, 3, 1, 6, 0, 2, 9])
    off = R.make_offsets(ln)
    x = rand(off[-1] * 5, 3).reshape(-1, 5)
    xr = bf16_round(x) if dtype == torch.bfloat16 else f32_round(x)
    X = jt(off, xr, dtype)
    for L, pad in [(9, -7.5), (4, 0.0), (12, float("-inf"))]:
        d = J.jagged_to_dense(X, L, pad)
        np.testing.assert_array_equal(d.double().cpu().numpy(), R.jagged_to_dense(off, xr, L, pad))
    back = J.dense_to_jagged(J.jagged_to_dense(X, 9, 1.25), ln)
    assert torch.equal(back.values, X.values)
    np.testing.assert_array_equal(back.host_offsets, off)
    s = rand(R.sum_sq(off), 4)
    sr = bf16_round(s) if dtype == torch.bfloat16 else f32_round(s)
    S = J.Jagged2Tensor(torch.from_numpy(off).to(DEV), torch.from_numpy(sr).to(dtype).to(DEV), off)
    for L in (9, 5):
        np.testing.assert_array_equal(J.jagged2_to_dense(S, L, -3.0).double().cpu().numpy(),
                                      R.jagged2_to_dense(off, sr, L, -3.0))
    S2 = J.dense_to_jagged2(J.jagged2_to_dense(S, 9, 0.0), ln)
    assert torch.equal(S2.values, S.values)
    with pytest.raises(J.JaggedError, match="dense_to_jagged: sample 6 length 9 exceeds max_len 8"):
        J.dense_to_jagged(torch.zeros(7, 8, 5, device=DEV), ln)


def test_elementwise_ops():
    ln = np.array([2, 0, 3])
    off = R.make_offsets(ln)
    a, b = f32_round(rand(20, 1)).reshape(5, 4), f32_round(rand(20, 2)).reshape(5, 4)
    A, B = jt(off, a), jt(off, b)
    for fn, ref in [(J.add, a + b), (J.sub, a - b), (J.mul, a * b)]:
        np.testing.assert_array_equal(fn(A, B).values.double().cpu().numpy(), f32_round(ref))
    np.testing.assert_array_equal(J.scale(A, 0.5).values.double().cpu().numpy(), a * 0.5)
    with pytest.raises(J.JaggedError, match="add: offsets differ first at sample 1"):
        J.add(A, jt(R.make_offsets([2, 1, 2]), b))
    with pytest.raises(J.JaggedError, match=r"sub: dim mismatch \(4 vs 2\)"):
        J.sub(A, jt(off, b[:, :2].copy()))


# ------------------------------------------------------------------ Table-1 operators (fp32 mode)
def _inputs(ln, D, T, seed, rnd):
    off = R.make_offsets(ln)
    S, B, SQ = int(off[-1]), len(ln), R.sum_sq(off)
    v = rnd(rand(3 * S * max(D, T) + 2 * SQ + 3 * B * D * T + S * (D + T), seed))
    c = [0]

    def take(n, shape):
        a = v[c[0]:c[0] + n].reshape(shape)
        c[0] += n
        return a
    return off, dict(x=take(S * D, (S, D)), y=take(S * T, (S, T)), k=take(S * D, (S, D)), w=take(B * D * T, (B, D, T)),
                     a=take(SQ, (SQ,)), go_t=take(S * T, (S, T)), go_d=take(S * D, (S, D)),
                     go_dt=take(B * D * T, (B, D, T)), go_sq=take(SQ, (SQ,)))


CASES = [("golden", 16, 8), ("uniform", 64, 32), ("long", 32, 48),
         ("long", 128, 64), ("golden", 64, 128), ("uniform", 256, 256)]  # the last three hit tcgen05 (bf16)


@pytest.mark.parametrize("lset,D,T", CASES)
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_table1_forward(lset, D, T, mode):
    ln = np.asarray(LENGTH_SETS[lset], np.int64)
    dtype = torch.float32 if mode == "fp32" else torch.bfloat16
    rnd = f32_round if mode == "fp32" else bf16_round
    close = assert_fp32_close if mode == "fp32" else assert_bf16_close
    off, t = _inputs(ln, D, T, 11, rnd)
    od = torch.float32
    X, Y, K = jt(off, t["x"], dtype), jt(off, t["y"], dtype), jt(off, t["k"], dtype)
    W = torch.from_numpy(t["w"]).to(dtype).to(DEV)
    close(J.jagged_dense_bmm(X, W, out_dtype=od).values, R.jagged_dense_bmm(off, t["x"], t["w"]), what="jdbmm")
    close(J.jagged_jagged_bmm(X, Y, out_dtype=od), R.jagged_jagged_bmm(off, t["x"], t["y"]), what="jjbmm")
    S = J.jagged_jagged_bmm_jagged_out(X, K, out_dtype=od)
    close(S.values, R.jagged_jagged_bmm_jagged_out(off, t["x"], t["k"]), what="jjbmm_jout")
    A = J.Jagged2Tensor(X.offsets, torch.from_numpy(t["a"]).to(dtype).to(DEV), off)
    close(J.array_jagged_bmm_jagged_out(A, X, out_dtype=od).values, R.array_jagged_bmm_jagged_out(off, t["a"], t["x"]),
          what="ajbmm_jout")
    # softmaxes (output dtype = input dtype; |p| <= 1 so bf16 output is within 2e-2)
    close(J.jagged_softmax(X).values, R.jagged_softmax(off, t["x"]), what="jagged_softmax")
    close(J.jagged2_softmax(A).values, R.jagged2_softmax(off, t["a"]), what="jagged2_softmax")


@pytest.mark.parametrize("lset,D,T", CASES)
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_table1_vjps(lset, D, T, mode):
    ln = np.asarray(LENGTH_SETS[lset], np.int64)
    dtype = torch.float32 if mode == "fp32" else torch.bfloat16
    rnd = f32_round if mode == "fp32" else bf16_round
    close = assert_fp32_close if mode == "fp32" else assert_bf16_close
    off, t = _inputs(ln, D, T, 12, rnd)
    od = torch.float32
    X, Y, K = jt(off, t["x"], dtype), jt(off, t["y"], dtype), jt(off, t["k"], dtype)
    W = torch.from_numpy(t["w"]).to(dtype).to(DEV)
    GT, GD = jt(off, t["go_t"], dtype), jt(off, t["go_d"], dtype)
    GDT = torch.from_numpy(t["go_dt"]).to(dtype).to(DEV)
    A = J.Jagged2Tensor(X.offsets, torch.from_numpy(t["a"]).to(dtype).to(DEV), off)
    GSQ = J.Jagged2Tensor(X.offsets, torch.from_numpy(t["go_sq"]).to(dtype).to(DEV), off)

    dx, dw = J.jagged_dense_bmm_vjp(X, W, GT, out_dtype=od)
    rx, rw = R.jagged_dense_bmm_vjp(off, t["x"], t["w"], t["go_t"])
    close(dx.values, rx, what="jdbmm dx"); close(dw, rw, what="jdbmm dw")
    dx, dy = J.jagged_jagged_bmm_vjp(X, Y, GDT, out_dtype=od)
    rx, ry = R.jagged_jagged_bmm_vjp(off, t["x"], t["y"], t["go_dt"])
    close(dx.values, rx, what="jjbmm dx"); close(dy.values, ry, what="jjbmm dy")
    dq, dk = J.jagged_jagged_bmm_jagged_out_vjp(X, K, GSQ, out_dtype=od)
    rq, rk = R.jagged_jagged_bmm_jagged_out_vjp(off, t["x"], t["k"], t["go_sq"])
    close(dq.values, rq, what="jjbmm_jout dq"); close(dk.values, rk, what="jjbmm_jout dk")
    da, dv = J.array_jagged_bmm_jagged_out_vjp(A, X, GD, out_dtype=od)
    ra, rv = R.array_jagged_bmm_jagged_out_vjp(off, t["a"], t["x"], t["go_d"])
    close(da.values, ra, what="ajbmm da"); close(dv.values, rv, what="ajbmm dv")
    close(J.jagged_softmax_vjp(X, GD).values, R.jagged_softmax_vjp(off, t["x"], t["go_d"]), what="jsoftmax vjp")
    close(J.jagged2_softmax_vjp(A, GSQ).values, R.jagged2_softmax_vjp(off, t["a"], t["go_sq"]), what="j2softmax vjp")


def test_golden_fixture_ops(golden):
    """The reference's own outputs (tests/golden/ops.npz) vs the GPU in fp32 mode."""
    o = golden["ops"]
    off = o["offsets"]
    X, Y, K = jt(off, o["x"]), jt(off, o["y"]), jt(off, o["k"])
    # inputs were binary64; the GPU sees them rounded to fp32, so compare at fp32 tolerance
    assert_fp32_close(J.jagged_dense_bmm(X, torch.from_numpy(o["w"]).float().to(DEV)).values,
                      o["jagged_dense_bmm"], tol=2e-5, what="jdbmm")
    assert_fp32_close(J.jagged_jagged_bmm(X, Y), o["jagged_jagged_bmm"], tol=2e-5, what="jjbmm")
    assert_fp32_close(J.jagged_softmax(X).values, o["jagged_softmax"], tol=2e-5, what="softmax")
    assert_fp32_close(J.jagged_jagged_bmm_jagged_out(X, K).values, o["jagged_jagged_bmm_jagged_out"], tol=2e-5)
    A = J.Jagged2Tensor(X.offsets, torch.from_numpy(o["a"]).float().to(DEV), off)
    assert_fp32_close(J.array_jagged_bmm_jagged_out(A, X).values, o["array_jagged_bmm_jagged_out"], tol=2e-5)
    assert_fp32_close(J.jagged2_softmax(A).values, o["jagged2_softmax"], tol=2e-5)


def test_known_answer_vectors(golden):
    kat = golden["kat"]
    X = jt(R.make_offsets([2, 1]), np.array([[1, 2], [3, 4], [5, 6]], np.float32))
    W = torch.tensor([[[1.0], [1.0]], [[2.0], [0.0]]], device=DEV)
    np.testing.assert_array_equal(J.jagged_dense_bmm(X, W).values.cpu().numpy().reshape(-1), kat["jdbmm_expect"])
    off1 = R.make_offsets([2])
    Z = J.jagged_jagged_bmm(jt(off1, np.eye(2, dtype=np.float32)), jt(off1, np.array([[2.0], [3.0]], np.float32)))
    np.testing.assert_array_equal(Z.cpu().numpy().reshape(-1), kat["jjbmm_expect"])
    sm = J.jagged_softmax(jt(off1, np.array([[0.0], [np.log(2)]], np.float32)))
    np.testing.assert_allclose(sm.values.cpu().numpy().reshape(-1), kat["jsoftmax_expect"], rtol=1e-6)
    A = J.Jagged2Tensor(torch.from_numpy(off1).to(DEV), torch.tensor([0, np.log(3), 0, 0], dtype=torch.float32,
                                                                        device=DEV), off1)
    np.testing.assert_allclose(J.jagged2_softmax(A).values.cpu().numpy(), kat["j2softmax_expect"], rtol=1e-6)
    one = J.jagged_softmax(jt(R.make_offsets([1]), np.array([[123.0, -7.0]], np.float32)))
    np.testing.assert_array_equal(one.values.cpu().numpy().reshape(-1), [1.0, 1.0])


def test_operator_errors_match_reference():
    off = R.make_offsets([2, 1])
    X = jt(off, np.zeros((3, 4), np.float32))
    with pytest.raises(J.JaggedError, match=r"jagged_dense_bmm: w must be \[B, D, T\]"):
        J.jagged_dense_bmm(X, torch.zeros(2, 4, device=DEV))
    with pytest.raises(J.JaggedError, match=r"jagged_dense_bmm: batch mismatch \(2 vs 3\)"):
        J.jagged_dense_bmm(X, torch.zeros(3, 4, 2, device=DEV))
    with pytest.raises(J.JaggedError, match=r"jagged_dense_bmm: dim mismatch \(4 vs 5\)"):
        J.jagged_dense_bmm(X, torch.zeros(2, 5, 2, device=DEV))
    Y = jt(R.make_offsets([1, 2]), np.zeros((3, 4), np.float32))
    with pytest.raises(J.JaggedError, match="jagged_jagged_bmm: offsets differ first at sample 0"):
        J.jagged_jagged_bmm(X, Y)
    A = J.Jagged2Tensor(Y.offsets, torch.zeros(5, device=DEV), Y.host_offsets)
    with pytest.raises(J.JaggedError, match="array_jagged_bmm_jagged_out: length mismatch at sample 0"):
        J.array_jagged_bmm_jagged_out(A, X)
    with pytest.raises(J.JaggedError, match="JaggedTensor: offsets must start with 0"):
        jt([1, 3], np.zeros((2, 1), np.float32))
    with pytest.raises(J.JaggedError, match="non-decreasing at index 2"):
        jt([0, 3, 2], np.zeros((2, 1), np.float32))
    with pytest.raises(J._lib.JaggedDeviceError, match="JG_UNSUPPORTED"):
        J.jagged_softmax(J.JaggedTensor(X.offsets, torch.zeros(3, 4, dtype=torch.float64, device=DEV), off))


def test_empty_samples_zero_dense_outputs():
    """jagged_jagged_bmm writes zeros for empty samples (linalg.cpp:75)."""
    ln = np.array([0, 3, 0])
    off = R.make_offsets(ln)
    X = jt(off, f32_round(rand(12, 5)).reshape(3, 4))
    Z = torch.full((3, 4, 4), 7.0, device=DEV)
    out = J.jagged_jagged_bmm(X, X)
    assert out.shape == (3, 4, 4) and bool((out[0] == 0).all()) and bool((out[2] == 0).all())
    del Z
    _, dw = J.jagged_dense_bmm_vjp(X, torch.ones(3, 4, 2, device=DEV), jt(off, np.ones((3, 2), np.float32)))
    assert bool((dw[0] == 0).all()) and bool((dw[2] == 0).all())


def test_full_size_cfg4_properties():
    """BASELINE cfg4 at full size (half-mean B=2048, L=1024 seed 0: sum_B = 1,048,576, SQ = 7.2461e8; D=T=256 bf16):
    size-independent identities that tie the Table-1 ops together, plus whole-sample fp32 spot checks.
      * per-sample associativity: (Q_i K_i^T) V_i == Q_i (K_i^T V_i), i.e.
        array_jagged_bmm_jagged_out(jagged_jagged_bmm_jagged_out(Q, K), V) == jagged_dense_bmm(Q, jagged_jagged_bmm(K, V))
      * softmax normalisation: jagged_softmax columns and jagged2_softmax rows sum to 1.
    bf16 inputs; tolerances relative to the magnitudes involved (bf16 rounding of the intermediates)."""
    ln = R.gen_lengths("half-mean", 1024, 0, 2048)
    off = R.make_offsets(ln)
    S, D = int(off[-1]), 256
    assert S == 1_048_576
    g = torch.Generator(device=DEV).manual_seed(5)
    r = lambda *sh: ((torch.rand(*sh, device=DEV, generator=g) * 2 - 1) * 0.25).bfloat16()  # noqa: E731
    offd = torch.from_numpy(off).to(DEV)
    Q, K, V = (J.JaggedTensor(offd, r(S, D), off) for _ in range(3))
    lhs = J.array_jagged_bmm_jagged_out(J.jagged_jagged_bmm_jagged_out(Q, K), V).values.float()
    rhs = J.jagged_dense_bmm(Q, J.jagged_jagged_bmm(K, V)).values.float()
    scale = float(rhs.abs().max())
    err = float((lhs - rhs).abs().max())
    assert err <= 2e-2 * scale, f"associativity: max |(QK^T)V - Q(K^T V)| = {err:.3e} vs max |.| = {scale:.3e}"
    # whole-sample fp32 spot checks (largest and a few others)
    nz = np.nonzero(ln)[0]
    for i in {int(nz[np.argmax(ln[nz])]), int(nz[0]), int(nz[len(nz) // 2])}:
        a, b = int(off[i]), int(off[i + 1])
        q, k, v = (t.values[a:b].float() for t in (Q, K, V))
        ref = (q @ k.T).bfloat16().float() @ v  # the jagged^2 intermediate is bf16, as in the device path
        assert_bf16_close(lhs[a:b], ref.cpu().numpy(), what=f"ajbmm(jjbmm_jout) sample {i} (n={b - a})")
    # softmax normalisation
    X = J.JaggedTensor(offd, r(S, D) * 8, off)
    P = J.jagged_softmax(X).values.float()
    seg = torch.repeat_interleave(torch.arange(len(ln), device=DEV), torch.from_numpy(ln).to(DEV))
    colsum = torch.zeros(len(ln), D, device=DEV).index_add_(0, seg, P)
    ne = torch.from_numpy(ln > 0).to(DEV)
    assert float((colsum[ne] - 1).abs().max()) < 2e-2 and bool((P >= 0).all())
    A = J.jagged_jagged_bmm_jagged_out(Q, K)
    P2 = J.jagged2_softmax(A)
    rows = torch.repeat_interleave(torch.from_numpy(ln).to(DEV), torch.from_numpy(ln).to(DEV))  # Bi per row
    row_id = torch.repeat_interleave(torch.arange(S, device=DEV), rows)
    rowsum = torch.zeros(S, device=DEV).index_add_(0, row_id, P2.values.float())
    assert float((rowsum - 1).abs().max()) < 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("lens", [[1, 7, 129, 300, 0, 255, 513, 8, 9, 1000], list(range(1, 140, 3)), [1024] * 4 + [1023] * 3])
def test_jjjout_bf16_output_matches_rounded_f32(lens):
    """bf16-output jagged_jagged_bmm_jagged_out (tcgen05 epilogue writing realigned bf16 row images, every
    row phase mod 8) equals the fp32-output run of the same kernel rounded to bf16 — bit for bit — and the
    f64 oracle within the bf16 tolerance plus the bf16 storage rounding."""
    ln = np.asarray(lens, np.int64)
    D = 128
    off, t = _inputs(ln, D, 8, 5, bf16_round)
    X, K = jt(off, t["x"], torch.bfloat16), jt(off, t["k"], torch.bfloat16)
    s32 = J.jagged_jagged_bmm_jagged_out(X, K, out_dtype=torch.float32).values
    s16 = J.jagged_jagged_bmm_jagged_out(X, K).values
    assert s16.dtype == torch.bfloat16 and s16.numel() == int((ln * ln).sum())
    assert torch.equal(s16, s32.bfloat16())
    ref = torch.from_numpy(np.asarray(R.jagged_jagged_bmm_jagged_out(off, t["x"], t["k"]), np.float64))
    assert_bf16_close(s32, ref, what="jjbmm_jout f32 out")
    # bf16 storage adds at most half an ulp (2^-9 relative) of the output's own magnitude
    err = (s16.double().cpu() - ref).abs()
    assert bool((err <= 2e-2 + ref.abs() * 2.0 ** -8).all()), float(err.max())
