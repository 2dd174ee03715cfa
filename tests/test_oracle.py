"""Pins the C restatement (oracle/jagged_oracle.c) before any GPU result is trusted.

Three anchors: the SPEC known-answer vectors, golden fixtures produced by the
compiled reference (tests/golden/make_golden.py), and — where oracle/_ref is present — a live
comparison with the reference on fresh inputs. All CPU-only.
"""
import numpy as np
import pytest

from oracle import reference as F
from oracle import restated as R

EXACT = dict(rtol=1e-13, atol=1e-15)


def test_rng_and_lengths_bit_exact(golden):
    ln = golden["lengths"]
    assert (R.gen_lengths("uniform", 128, 0, 64) == ln["cfg1_uniform_B64_L128"]).all()
    assert (R.gen_lengths("half-mean", 1024, 0, 1024) == ln["cfg3_halfmean_B1024_L1024"]).all()
    assert (R.gen_lengths("half-mean", 1024, 0, 2048) == ln["cfg4_halfmean_B2048_L1024"]).all()
    assert (R.gen_lengths("uniform", 50, 9, 33) == ln["uniform_B33_L50_s9"]).all()
    assert (R.gen_lengths("half-mean", 50, 9, 33) == ln["halfmean_B33_L50_s9"]).all()
    # sizes quoted in SURVEY.md §8(d) / P4
    assert R.gen_lengths("uniform", 128, 0, 64).sum() == 3604
    h = R.gen_lengths("half-mean", 1024, 0, 1024)
    assert h.sum() == 524288 and (h * h).sum() == 362240860 and (h == 0).sum() == 2
    assert R.gen_lengths("half-mean", 1024, 0, 2048).sum() == 1048576
    z = R.gen_lengths("zipf", 512, 0, 256, 1.1)
    assert z.sum() == 15676 and int(np.median(z)) == 14 and z.max() == 498


def test_fixed_and_errors():
    assert (R.gen_lengths("fixed", 7, 3, 5) == 7).all()
    with pytest.raises(R.OracleError, match="batch must be >= 1"):
        R.gen_lengths("uniform", 7, 0, 0)
    with pytest.raises(R.OracleError, match="negative length at sample 1"):
        R.make_offsets([3, -1, 2])


def test_known_answer_vectors(golden):
    kat = golden["kat"]
    off = R.make_offsets([2, 1])
    x = np.array([[1, 2], [3, 4], [5, 6]], float)
    w = np.array([[[1], [1]], [[2], [0]]], float)
    np.testing.assert_array_equal(R.jagged_dense_bmm(off, x, w).reshape(-1), kat["jdbmm_expect"])
    off1 = R.make_offsets([2])
    np.testing.assert_array_equal(R.jagged_jagged_bmm(off1, np.eye(2), [[2.0], [3.0]]).reshape(-1),
                                  kat["jjbmm_expect"])
    np.testing.assert_allclose(R.jagged_softmax(off1, [[0.0], [np.log(2)]]).reshape(-1), kat["jsoftmax_expect"],
                               rtol=1e-15)
    np.testing.assert_allclose(R.jagged2_softmax(off1, [0, np.log(3), 0, 0]), kat["j2softmax_expect"], rtol=1e-15)
    # the reference's own outputs on the same KATs
    for key in ("jdbmm", "jjbmm", "jsoftmax", "j2softmax"):
        np.testing.assert_allclose(kat[key + "_out"], kat[key + "_expect"], rtol=1e-15)
    np.testing.assert_array_equal(R.jagged_softmax(R.make_offsets([1]), [[123.0, -7.0]]).reshape(-1),
                                  kat["jsoftmax_single"])


def test_operators_vs_reference_golden(golden):
    o = golden["ops"]
    off = o["offsets"]
    chk = lambda a, b: np.testing.assert_allclose(a, b, **EXACT)  # noqa: E731
    chk(R.jagged_dense_bmm(off, o["x"], o["w"]), o["jagged_dense_bmm"])
    chk(R.jagged_jagged_bmm(off, o["x"], o["y"]), o["jagged_jagged_bmm"])
    chk(R.jagged_softmax(off, o["x"]), o["jagged_softmax"])
    chk(R.jagged_jagged_bmm_jagged_out(off, o["x"], o["k"]), o["jagged_jagged_bmm_jagged_out"])
    chk(R.array_jagged_bmm_jagged_out(off, o["a"], o["x"]), o["array_jagged_bmm_jagged_out"])
    chk(R.jagged2_softmax(off, o["a"]), o["jagged2_softmax"])
    dx, dw = R.jagged_dense_bmm_vjp(off, o["x"], o["w"], o["go_t"])
    chk(dx, o["jagged_dense_bmm_vjp_dx"]); chk(dw, o["jagged_dense_bmm_vjp_dw"])
    dx, dy = R.jagged_jagged_bmm_vjp(off, o["x"], o["y"], o["go_dt"])
    chk(dx, o["jagged_jagged_bmm_vjp_dx"]); chk(dy, o["jagged_jagged_bmm_vjp_dy"])
    chk(R.jagged_softmax_vjp(off, o["x"], o["go_d"]), o["jagged_softmax_vjp"])
    dq, dk = R.jagged_jagged_bmm_jagged_out_vjp(off, o["x"], o["k"], o["go_sq"])
    chk(dq, o["jjbmm_jout_vjp_dq"]); chk(dk, o["jjbmm_jout_vjp_dk"])
    da, dv = R.array_jagged_bmm_jagged_out_vjp(off, o["a"], o["x"], o["go_d"])
    chk(da, o["ajbmm_jout_vjp_da"]); chk(dv, o["ajbmm_jout_vjp_dv"])
    chk(R.jagged2_softmax_vjp(off, o["a"], o["go_sq"]), o["jagged2_softmax_vjp"])


def test_attention_vs_reference_golden(golden):
    a = golden["attention"]
    off = a["offsets"]
    np.testing.assert_allclose(R.jagged_attention(off, a["q"], a["k"], a["v"]), a["jagged_attention"], **EXACT)
    for bq, bk in [(3, 3), (64, 64)]:
        tag = f"b{bq}x{bk}"
        out, lse = R.jfa_forward(off, a["q"], a["k"], a["v"], bq, bk)
        np.testing.assert_allclose(out, a[f"out_{tag}"], **EXACT)
        np.testing.assert_array_equal(np.isinf(lse), np.isinf(a[f"lse_{tag}"]))
        fin = np.isfinite(lse)
        np.testing.assert_allclose(lse[fin], a[f"lse_{tag}"][fin], **EXACT)
        dq, dk, dv = R.jfa_backward(off, a["q"], a["k"], a["v"], a["go"], out, lse, bk)
        np.testing.assert_allclose(dq, a[f"dq_{tag}"], **EXACT)
        np.testing.assert_allclose(dk, a[f"dk_{tag}"], **EXACT)
        np.testing.assert_allclose(dv, a[f"dv_{tag}"], **EXACT)


def test_attention_invariants(golden):
    """unfused == flash, lse matches the naive path, convexity, empty segments."""
    a = golden["attention"]
    off = a["offsets"]
    out, lse = R.jfa_forward(off, a["q"], a["k"], a["v"], 64, 64)
    np.testing.assert_allclose(out, R.jagged_attention(off, a["q"], a["k"], a["v"]), rtol=1e-9, atol=1e-12)
    ln = np.diff(off)
    assert np.isinf(lse[off[0]:off[1]]).all() if ln[0] else True
    for i in range(len(ln)):
        if ln[i] == 0:
            continue
        seg = slice(off[i], off[i + 1])
        vmin, vmax = a["v"][seg].min(0), a["v"][seg].max(0)
        assert (out[seg] >= vmin - 1e-9).all() and (out[seg] <= vmax + 1e-9).all()
    # padded dense attention restricted to valid rows == jagged
    L = int(ln.max())
    qp, kp, vp = (R.jagged_to_dense(off, t, L) for t in (a["q"], a["k"], a["v"]))
    dense = R.dense_attention(ln, qp, kp, vp)
    np.testing.assert_allclose(R.dense_to_jagged(dense, ln), out, rtol=1e-9, atol=1e-12)


def test_layout_roundtrip():
    rng = R.Rng(3)
    ln = np.array([0, 3, 1, 6, 0, 2])
    off = R.make_offsets(ln)
    x = rng.uniform_values(off[-1] * 4).reshape(-1, 4)
    d = R.jagged_to_dense(off, x, 6, pad=-7.5)
    np.testing.assert_array_equal(R.dense_to_jagged(d, ln), x)
    assert (d[0] == -7.5).all() and (d[2, 1:] == -7.5).all()
    t = R.jagged_to_dense(off, x, 2)  # truncation (tensor.cpp:108)
    np.testing.assert_array_equal(t[3], x[off[3]:off[3] + 2])
    s = rng.uniform_values(R.sum_sq(off))
    np.testing.assert_array_equal(R.dense_to_jagged2(R.jagged2_to_dense(off, s, 6, 9.0), ln), s)
    with pytest.raises(R.OracleError, match="sample 3 length 6 exceeds max_len 5"):
        R.dense_to_jagged(np.zeros((6, 5, 4)), ln)


@pytest.mark.skipif(not F.available(), reason="oracle/_ref not built")
def test_live_reference_random_shapes():
    """Fresh inputs through both the compiled reference and the restatement (uniform lengths)."""
    for seed in (1, 2):
        ln = R.gen_lengths("uniform", 40, seed, 9)
        ln[seed] = 0
        off = R.make_offsets(ln)
        D = 12
        vals = R.Rng(seed + 100).uniform_values(4 * off[-1] * D, as_float=False)
        q, k, v, go = (vals[i * off[-1] * D:(i + 1) * off[-1] * D].reshape(-1, D) for i in range(4))
        o1, l1 = R.jfa_forward(off, q, k, v, 5, 7)
        o2, l2 = F.jfa_forward(off, q, k, v, 5, 7)
        np.testing.assert_allclose(o1, o2, **EXACT)
        g1 = R.jfa_backward(off, q, k, v, go, o1, l1, 7)
        g2 = F.jfa_backward(off, q, k, v, go, o2, l2, 5, 7)
        for a_, b_ in zip(g1, g2):
            np.testing.assert_allclose(a_, b_, **EXACT)
        np.testing.assert_allclose(R.jagged_softmax(off, q), F.jagged_softmax(off, q), **EXACT)


def _mlp_layers(nx):
    return [(nx["mlp_w0"], nx["mlp_b0"], True), (nx["mlp_w1"], nx["mlp_b1"], False)]


def test_next_rows_vs_reference_golden(golden):
    """SURVEY §8f-1 feature_interaction and §8f-2 jagged_mlp (+VJP): oracle vs the reference's outputs."""
    nx = golden["next"]
    fi = R.feature_interaction(nx["fi_off"], nx["fi_k"], nx["fi_v"], nx["fi_targets"])
    np.testing.assert_allclose(fi, nx["fi_out_f64"], rtol=1e-12, atol=1e-14)
    # float instantiation: the oracle's as_float mode rounds where the reference's composed ops do
    fi32 = R.feature_interaction(nx["fi_off"], nx["fi_k"].astype(np.float32), nx["fi_v"].astype(np.float32),
                                 nx["fi_targets"].astype(np.float32), as_float=True)
    np.testing.assert_allclose(fi32, nx["fi_out_f32"], rtol=2e-6, atol=1e-7)
    layers = _mlp_layers(nx)
    np.testing.assert_allclose(R.jagged_mlp(nx["mlp_x"], layers), nx["mlp_out_f64"], rtol=1e-12, atol=1e-13)
    dx, g = R.jagged_mlp_vjp(nx["mlp_x"], layers, nx["mlp_go"])
    np.testing.assert_allclose(dx, nx["mlp_dx"], rtol=1e-12, atol=1e-13)
    for l, (dw, db) in enumerate(g):
        np.testing.assert_allclose(dw, nx[f"mlp_dw{l}"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(db, nx[f"mlp_db{l}"], rtol=1e-12, atol=1e-13)
    with pytest.raises(R.OracleError, match="at least one layer"):
        R._chk(R.lib().or_jagged_mlp(1, 0, np.zeros(1, np.int64), np.zeros(1), np.zeros(1), None, np.zeros(1),
                                     np.zeros(1)))


@pytest.mark.skipif(not F.available(), reason="oracle/_ref not built")
def test_next_rows_live_reference():
    rng = np.random.default_rng(5)
    for lens, D, Tq in (([3, 0, 9, 1], 8, 5), ([40, 2, 0, 17, 63], 32, 2)):
        off = F.make_offsets(lens)
        S = int(off[-1])
        k, v = rng.uniform(-1, 1, (S, D)), rng.uniform(-1, 1, (S, D))
        tg = rng.uniform(-1, 1, (len(lens), Tq, D))
        np.testing.assert_allclose(R.feature_interaction(off, k, v, tg), F.feature_interaction(off, k, v, tg),
                                   rtol=1e-12, atol=1e-14)
    rows, dims = 19, [5, 7, 3, 4]
    x = rng.uniform(-1, 1, (rows, dims[0]))
    layers = [(rng.uniform(-1, 1, (dims[l], dims[l + 1])), rng.uniform(-1, 1, dims[l + 1]), l % 2 == 0)
              for l in range(3)]
    go = rng.uniform(-1, 1, (rows, dims[-1]))
    np.testing.assert_allclose(R.jagged_mlp(x, layers), F.jagged_mlp(x, layers), rtol=1e-12, atol=1e-13)
    dx, g = R.jagged_mlp_vjp(x, layers, go)
    rdx, rg = F.jagged_mlp_vjp(x, layers, go)
    np.testing.assert_allclose(dx, rdx, rtol=1e-12, atol=1e-13)
    for (a, b), (c, d) in zip(g, rg):
        np.testing.assert_allclose(a, c, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(b, d, rtol=1e-12, atol=1e-13)


def test_dense_flash_vs_reference_golden(golden):
    """SURVEY §8f-4 padded dense_flash_attention: oracle vs the reference's outputs (incl. a zero-length sample:
    zero rows and lse = -inf, attention.cpp:151-154)."""
    nx = golden["next"]
    ln, q, k, v = nx["df_len"], nx["df_q"], nx["df_k"], nx["df_v"]
    for bq, bk in ((3, 4), (64, 64)):
        o, lse = R.dense_flash_attention(ln, q, k, v, bq, bk)
        np.testing.assert_allclose(o, nx[f"df_out_f64_{bq}_{bk}"], rtol=1e-12, atol=1e-14)
        ref = nx[f"df_lse_f64_{bq}_{bk}"]
        assert np.array_equal(np.isinf(lse), np.isinf(ref))
        np.testing.assert_allclose(lse[np.isfinite(ref)], ref[np.isfinite(ref)], rtol=1e-12)
    # the f32 instantiation accumulates in double and rounds the outputs
    o32, l32 = R.dense_flash_attention(ln, *(a.astype(np.float32) for a in (q, k, v)))
    np.testing.assert_allclose(o32, nx["df_out_f32"], rtol=2e-6, atol=1e-7)
    fin = np.isfinite(nx["df_lse_f32"])
    np.testing.assert_allclose(l32[fin], nx["df_lse_f32"][fin], rtol=2e-6)
    # padded rows are zero; valid rows equal the unmasked dense attention
    np.testing.assert_allclose(o, R.dense_attention(ln, q, k, v), rtol=1e-12, atol=1e-14)
    with pytest.raises(R.OracleError):
        R._chk(R.lib().or_dense_flash_attention(ln, len(ln), q.shape[1], q.shape[2], 0, 4, q.reshape(-1),
                                                k.reshape(-1), v.reshape(-1), np.empty(q.size), np.empty(q.size)))


@pytest.mark.skipif(not F.available(), reason="oracle/_ref not built")
def test_dense_flash_live_reference():
    rng = np.random.default_rng(9)
    for ln, L, D, bq, bk in (([7, 0, 12, 12], 12, 16, 5, 3), ([1, 33, 20], 40, 8, 64, 64)):
        q, k, v = (rng.uniform(-1, 1, (len(ln), L, D)) for _ in range(3))
        o, lse = R.dense_flash_attention(ln, q, k, v, bq, bk)
        ro, rl = F.dense_flash_attention(ln, q, k, v, bq, bk)
        np.testing.assert_allclose(o, ro, rtol=1e-12, atol=1e-14)
        assert np.array_equal(np.isinf(lse), np.isinf(rl))
        np.testing.assert_allclose(lse[np.isfinite(rl)], rl[np.isfinite(rl)], rtol=1e-12)
