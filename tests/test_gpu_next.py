"""GPU parity of the SURVEY §8f "next" rows through the C-ABI: feature_interaction (attention.cpp:291-309)
and jagged_mlp forward + VJP (linalg.cpp:246-277, :509-573), against the binary64 oracle (pinned to the
reference by tests/test_oracle.py::test_next_rows_*) and the committed reference outputs (next.npz).
fp32 mode: 1e-5 relative; bf16 inputs: 2e-2 max-abs.
"""
import numpy as np
import pytest
import torch

from oracle import restated as R
from tests.parity import assert_bf16_close, assert_fp32_close, bf16_round, f32_round

pytestmark = pytest.mark.gpu
J = pytest.importorskip("paper_2409_15373_b200.jagged")
DEV = "cuda"


def jt(off, vals, dtype):
    off = np.asarray(off, np.int64)
    return J.JaggedTensor(torch.from_numpy(off).to(DEV), torch.from_numpy(np.asarray(vals)).to(dtype).to(DEV), off)


def dev(a, dtype):
    return torch.from_numpy(np.asarray(a)).to(dtype).to(DEV)


# ------------------------------------------------------------------ feature interaction
def test_feature_interaction_golden(golden):
    nx = golden["next"]
    off = nx["fi_off"]
    k, v, tg = (f32_round(nx[n]) for n in ("fi_k", "fi_v", "fi_targets"))
    out = J.feature_interaction(jt(off, k, torch.float32), jt(off, v, torch.float32), dev(tg, torch.float32))
    assert_fp32_close(out, nx["fi_out_f32"].astype(np.float64), what="fi vs reference f32")
    assert_fp32_close(out, R.feature_interaction(off, k, v, tg, as_float=True), what="fi vs oracle")
    # empty samples give zeros
    ln = np.diff(off)
    assert not out[torch.from_numpy(ln == 0).to(DEV)].any()


@pytest.mark.parametrize("lens,D,Tq", [([3, 0, 9, 1, 130, 64], 32, 5), ([257, 0, 70, 1, 128], 64, 64),
                                       (list(R.gen_lengths("uniform", 128, 0, 64)), 64, 32),
                                       ([5, 0, 300, 129, 0], 128, 300)])  # bf16 D=64/128: fused kernel
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_feature_interaction_random(lens, D, Tq, mode):
    off = R.make_offsets(lens)
    S, B = int(off[-1]), len(lens)
    vals = R.Rng(21).uniform_values(2 * S * D + B * Tq * D)
    rnd = f32_round if mode == "fp32" else bf16_round
    dtype = torch.float32 if mode == "fp32" else torch.bfloat16
    k, v = rnd(vals[:S * D].reshape(S, D)), rnd(vals[S * D:2 * S * D].reshape(S, D))
    tg = rnd(vals[2 * S * D:].reshape(B, Tq, D))
    out = J.feature_interaction(jt(off, k, dtype), jt(off, v, dtype), dev(tg, dtype))
    ref = R.feature_interaction(off, k, v, tg, as_float=True)
    if mode == "fp32":
        assert_fp32_close(out, ref, what="fi")
    else:
        assert_bf16_close(out, ref, what="fi bf16")


def test_feature_interaction_errors():
    off = R.make_offsets([2, 3])
    x = jt(off, np.zeros((5, 4)), torch.float32)
    y = jt(off, np.zeros((5, 3)), torch.float32)
    with pytest.raises(J.JaggedError, match="k_feat/v_feat layout mismatch"):
        J.feature_interaction(x, y, torch.zeros(2, 1, 4, device=DEV))
    with pytest.raises(J.JaggedError, match=r"targets must be \[B, Tq, D\]"):
        J.feature_interaction(x, x, torch.zeros(3, 1, 4, device=DEV))


# ------------------------------------------------------------------ jagged MLP
def _layers_dev(layers, dtype):
    return [J.MlpLayer(dev(w, dtype), dev(b, dtype), J.RELU if r else J.NONE) for w, b, r in layers]


def test_jagged_mlp_golden(golden):
    nx = golden["next"]
    layers = [(nx["mlp_w0"], nx["mlp_b0"], True), (nx["mlp_w1"], nx["mlp_b1"], False)]
    lf = [(f32_round(w), f32_round(b), r) for w, b, r in layers]
    x, go = f32_round(nx["mlp_x"]), f32_round(nx["mlp_go"])
    off = np.array([0, 10, 10, x.shape[0]], np.int64)   # the MLP ignores sample boundaries
    out = J.jagged_mlp(jt(off, x, torch.float32), _layers_dev(lf, torch.float32))
    assert_fp32_close(out.values, nx["mlp_out_f32"].astype(np.float64), what="mlp vs reference f32")
    assert_fp32_close(out.values, R.jagged_mlp(x, lf), what="mlp vs oracle")
    g = J.jagged_mlp_vjp(jt(off, x, torch.float32), _layers_dev(lf, torch.float32), jt(off, go, torch.float32))
    dx, rg = R.jagged_mlp_vjp(x, lf, go)
    assert_fp32_close(g.dx.values, dx, what="dx")
    for l, (dw, db) in enumerate(rg):
        assert_fp32_close(g.dlayers[l].dweights, dw, what=f"dW{l}")
        assert_fp32_close(g.dlayers[l].dbias, db, what=f"db{l}")


@pytest.mark.parametrize("rows,dims", [(1000, [64, 128, 64]), (4099, [128, 64, 192, 64]), (0, [16, 8])])
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_jagged_mlp_random(rows, dims, mode):
    rng = R.Rng(33)
    rnd = f32_round if mode == "fp32" else bf16_round
    dtype = torch.float32 if mode == "fp32" else torch.bfloat16
    # weights scaled by 1/sqrt(d_in) keep activations O(1) (bf16 keeps ~3 significant digits). In bf16 only the
    # first layer is ReLU: deeper pre-activations differ from the binary64 chain by bf16 rounding, so ReLU masks
    # flip wherever |pre-activation| < ~1e-2 and the gradient difference there is O(1) by construction.
    relu = [(l == 0) if mode == "bf16" else (l % 2 == 0) for l in range(len(dims) - 1)]
    layers = [(rnd(rng.uniform_values(dims[l] * dims[l + 1]).reshape(dims[l], dims[l + 1]) / np.sqrt(dims[l])),
               rnd(rng.uniform_values(dims[l + 1]) * 0.1), relu[l]) for l in range(len(dims) - 1)]
    x = rnd(rng.uniform_values(rows * dims[0]).reshape(rows, dims[0]))
    go = rnd(rng.uniform_values(rows * dims[-1]).reshape(rows, dims[-1]))
    off = np.array([0, rows // 3, rows], np.int64)
    L = _layers_dev(layers, dtype)
    out = J.jagged_mlp(jt(off, x, dtype), L)
    g = J.jagged_mlp_vjp(jt(off, x, dtype), L, jt(off, go, dtype))
    ref = R.jagged_mlp(x, layers)
    dx, rg = R.jagged_mlp_vjp(x, layers, go)
    if mode == "fp32":
        assert_fp32_close(out.values, ref, what="mlp")
        assert_fp32_close(g.dx.values, dx, what="dx")
        for l, (dw, db) in enumerate(rg):
            assert_fp32_close(g.dlayers[l].dweights, dw, what=f"dW{l}")
            assert_fp32_close(g.dlayers[l].dbias, db, what=f"db{l}")
    else:
        assert_bf16_close(out.values, ref, what="mlp bf16")
        assert_bf16_close(g.dx.values, dx, what="dx bf16")
        for l, (dw, db) in enumerate(rg):
            # dW/db sum over all rows: compare relative to the reduction length (bf16 output rounding)
            scale = max(1.0, float(np.abs(dw).max()), float(np.abs(db).max()))
            assert_bf16_close(g.dlayers[l].dweights / scale, dw / scale, what=f"dW{l} bf16")
            assert_bf16_close(g.dlayers[l].dbias / scale, db / scale, what=f"db{l} bf16")


def test_jagged_mlp_errors():
    off = np.array([0, 2], np.int64)
    x = jt(off, np.zeros((2, 4)), torch.float32)
    with pytest.raises(J.JaggedError, match="at least one layer required"):
        J.jagged_mlp(x, [])
    with pytest.raises(J.JaggedError, match=r"layer 0 input dim mismatch \(4 vs 3\)"):
        J.jagged_mlp(x, [J.MlpLayer(torch.zeros(3, 2, device=DEV), torch.zeros(2, device=DEV))])
    with pytest.raises(J.JaggedError, match="layer 0 bias size 3 != 2"):
        J.jagged_mlp(x, [J.MlpLayer(torch.zeros(4, 2, device=DEV), torch.zeros(3, device=DEV))])
