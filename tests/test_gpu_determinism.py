"""Bit-identical attention gradients (the reference's fixed summation order,
attention.cpp:252-254): the tcgen05 backward accumulates the key tiles' partial dQ of every query block in 64-bit
fixed point, whose integer adds are order-independent, so dq/dk/dv must be torch.equal across repeated runs,
across grid sizes (a capped persistent grid changes which CTA runs which tile and in which order the tiles
arrive at a block); the fp32 mode (deterministic=False) agrees to rounding. Also checks the
results against the oracle so an ordering bug cannot hide behind self-consistency."""
import os

import numpy as np
import pytest
import torch

from oracle import reference as REF
from oracle import restated as R
from tests.parity import assert_bf16_close

pytestmark = pytest.mark.gpu
J = pytest.importorskip("paper_2409_15373_b200.jagged")
DEV = "cuda"


def _inputs(ln, H, D, seed):
    off = R.make_offsets(np.asarray(ln, np.int64))
    S = int(off[-1])
    vals = torch.from_numpy(R.Rng(seed).uniform_values(4 * S * H * D)).to(torch.bfloat16).reshape(4, S, H, D)
    return off, [J.JaggedTensor(torch.from_numpy(off).to(DEV), vals[i].to(DEV), off) for i in range(4)]


def _bwd(Q, K, V, G, saved, env=None, deterministic=True):
    old = {k: os.environ.get(k) for k in (env or {})}
    try:
        for k, v in (env or {}).items():
            os.environ[k] = v
        g = J.jagged_flash_attention_backward(Q, K, V, G, saved, deterministic=deterministic)
        torch.cuda.synchronize()
        return g
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


CASES = [
    (list(R.gen_lengths("half-mean", 1024, 0, 96)), 4, 128),          # cfg3-like: 1..8 key tiles per sample
    ([4092, 3000, 130, 1, 0, 257, 2048, 64, 129], 1, 128),             # up to 32 key tiles (cfg5-like)
    (list(R.gen_lengths("half-mean", 600, 3, 40)), 2, 64),
]


@pytest.mark.parametrize("ln,H,D", CASES)
def test_backward_bit_identical(ln, H, D):
    off, (Q, K, V, G) = _inputs(ln, H, D, 11)
    saved = J.jagged_flash_attention_forward(Q, K, V)
    ref = _bwd(Q, K, V, G, saved)
    variants = [
        {},                                   # repeat
        {},                                   # repeat
        {"JG_BWD_MAX_CTAS": "7"},             # smaller persistent grids: other CTAs, other arrival orders
        {"JG_BWD_MAX_CTAS": "61"},
    ]
    for env in variants:
        g = _bwd(Q, K, V, G, saved, env)
        for a, b, nm in ((g.dq, ref.dq, "dq"), (g.dk, ref.dk, "dk"), (g.dv, ref.dv, "dv")):
            assert torch.equal(a.values, b.values), f"{nm} differs under {env}"
    # fp32 accumulation (deterministic=False): dK/dV are unaffected (accumulated in TMEM in a fixed block order)
    # and dQ agrees to accumulation rounding
    g = _bwd(Q, K, V, G, saved, deterministic=False)
    assert torch.equal(g.dk.values, ref.dk.values) and torch.equal(g.dv.values, ref.dv.values)
    torch.testing.assert_close(g.dq.values.float(), ref.dq.values.float(), rtol=1e-2, atol=1e-3)
    # and it is the right answer: the compiled reference on a few samples (the longest included), head 0
    sub = sorted(set([i for i in range(len(ln)) if ln[i] > 0][:4]) | {int(np.argmax(ln))})
    idx = np.concatenate([np.arange(off[i], off[i + 1]) for i in sub])
    off_s = R.make_offsets(np.asarray(ln)[sub])
    qd, kd, vd, gd = (t.values[:, 0].double().cpu().numpy()[idx] for t in (Q, K, V, G))
    o_r, l_r = REF.jfa_forward(off_s, qd, kd, vd, 64, 64, prec="f64", threads=REF.hardware_threads())
    dq, dk, dv = REF.jfa_backward(off_s, qd, kd, vd, gd, o_r, l_r, 64, 64, prec="f64", threads=REF.hardware_threads())
    for got, r, nm in ((ref.dq, dq, "dq"), (ref.dk, dk, "dk"), (ref.dv, dv, "dv")):
        assert_bf16_close(got.values[:, 0].double().cpu().numpy()[idx], r, what=nm)
