"""GPU checks of the boundary's guards and edge semantics (advisor findings, round 1):

* -inf scores: the reference subtracts a finite max, so -inf entries get weight 0 while the rest of the
  column/row is a proper softmax (linalg.cpp:98-120, :199-220); an all -inf column is NaN in the reference
  (exp(-inf - -inf)) and stays NaN here.
* a caller-supplied schedule built for other offsets is rejected before any kernel reads it;
* paired operands must share dtype and device (the C-ABI takes one dtype);
* feature_interaction with every sample empty returns [B, Tq, D] zeros;
* repeated launches reuse the schedule's self-resetting work counters.
"""
import numpy as np
import pytest
import torch

from oracle import restated as R

pytestmark = pytest.mark.gpu
J = pytest.importorskip("paper_2409_15373_b200.jagged")
DEV = "cuda"


def jt(ln, vals, dtype=torch.float32):
    off = R.make_offsets(np.asarray(ln, np.int64))
    return J.JaggedTensor(torch.from_numpy(off).to(DEV), torch.as_tensor(vals).to(dtype).to(DEV), off)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_softmax_neg_inf_entries(dtype):
    ln = [5, 40, 3, 1]
    off = R.make_offsets(ln)
    x = R.Rng(4).uniform_values(int(off[-1]) * 64).reshape(-1, 64)
    x = torch.from_numpy(x).to(dtype).double().numpy()
    # -inf at the start of segments / columns (the running max starts at -inf), scattered -inf elsewhere
    x[0:2, :] = -np.inf
    x[5:25, 3] = -np.inf
    x[45:47, 7] = -np.inf
    x[10, :] = -np.inf
    X = jt(ln, x, dtype)
    got = J.jagged_softmax(X).values.double().cpu().numpy()
    ref = R.jagged_softmax(off, x)
    assert np.isfinite(ref).all()
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    assert np.isfinite(got).all(), "NaN from -inf entries"
    assert float(np.abs(got - ref).max()) <= tol
    # jagged2_softmax: -inf leading entries of rows
    s = R.Rng(5).uniform_values(int(sum(n * n for n in ln)))
    s = torch.from_numpy(s).to(dtype).double().numpy()
    s[0:3] = -np.inf                       # row 0 of block 0 starts with -inf
    s[25:25 + 39] = -np.inf                # row 0 of block 1: all but its last element
    S2 = J.Jagged2Tensor(X.offsets, torch.from_numpy(s).to(dtype).to(DEV), off)
    got2 = J.jagged2_softmax(S2).values.double().cpu().numpy()
    ref2 = R.jagged2_softmax(off, s)
    assert np.isfinite(ref2).all() and np.isfinite(got2).all()
    assert float(np.abs(got2 - ref2).max()) <= tol


def test_softmax_all_neg_inf_column_is_nan_like_reference():
    x = np.zeros((4, 32))
    x[:, 5] = -np.inf
    ref = R.jagged_softmax(R.make_offsets([4]), x)
    got = J.jagged_softmax(jt([4], x)).values.cpu().numpy()
    assert np.isnan(ref[:, 5]).all() and np.isnan(got[:, 5]).all()
    np.testing.assert_allclose(got[:, :5], ref[:, :5], rtol=1e-6)


def test_schedule_for_other_offsets_rejected():
    a = jt([100, 30, 200], np.zeros((330, 2, 64)), torch.bfloat16)
    b = jt([10, 20], np.zeros((30, 2, 64)), torch.bfloat16)
    sched_b = J.Schedule(b)
    with pytest.raises(J.JaggedError, match="schedule was built for other offsets"):
        J.jagged_flash_attention_forward(a, a, a, schedule=sched_b)
    saved = J.jagged_flash_attention_forward(a, a, a)
    with pytest.raises(J.JaggedError, match="schedule was built for other offsets"):
        J.jagged_flash_attention_backward(a, a, a, a, saved, schedule=sched_b)


def test_operand_dtype_and_device_checks():
    x = jt([3, 4], np.ones((7, 64)), torch.float32)
    w16 = torch.ones(2, 64, 32, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(J.JaggedError, match="dtype mismatch"):
        J.jagged_dense_bmm(x, w16)
    with pytest.raises(J.JaggedError, match="CUDA tensors"):
        J.jagged_dense_bmm(x, torch.ones(2, 64, 32))
    q = jt([3, 4], np.ones((7, 1, 64)), torch.float32)
    k16 = jt([3, 4], np.ones((7, 1, 64)), torch.bfloat16)
    with pytest.raises(J.JaggedError, match="dtype mismatch"):
        J.jagged_flash_attention_forward(q, k16, q)
    saved = J.jagged_flash_attention_forward(q, q, q)
    saved.logsumexp = saved.logsumexp.double()
    with pytest.raises(J.JaggedError, match="logsumexp must be a contiguous float32"):
        J.jagged_flash_attention_backward(q, q, q, q, saved)
    saved = J.jagged_flash_attention_forward(q, q, q)
    with pytest.raises(J.JaggedError, match="workspace needs"):
        J.jagged_flash_attention_backward(q, q, q, q, saved, workspace=torch.empty(16, dtype=torch.uint8, device=DEV))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_feature_interaction_all_empty(dtype):
    B, Tq, D = 3, 5, 64
    k = jt([0, 0, 0], np.zeros((0, D)), dtype)
    t = torch.ones(B, Tq, D, dtype=dtype, device=DEV)
    out = J.feature_interaction(k, k, t)
    assert out.shape == (B, Tq, D) and float(out.abs().max()) == 0.0


def test_repeated_launches_reuse_counters():
    """Many forward/backward launches through one schedule (self-resetting work counters) give identical
    results to fresh per-call schedules."""
    ln = list(R.gen_lengths("half-mean", 700, 2, 60))
    off = R.make_offsets(ln)
    S, H, D = int(off[-1]), 2, 128
    vals = torch.from_numpy(R.Rng(8).uniform_values(4 * S * H * D)).to(torch.bfloat16).reshape(4, S, H, D)
    Q, K, V, G = (J.JaggedTensor(torch.from_numpy(off).to(DEV), vals[i].to(DEV), off) for i in range(4))
    sched = J.Schedule(Q)
    ref = J.jagged_flash_attention_forward(Q, K, V)
    ref_g = J.jagged_flash_attention_backward(Q, K, V, G, ref)
    for _ in range(5):
        s = J.jagged_flash_attention_forward(Q, K, V, schedule=sched)
        g = J.jagged_flash_attention_backward(Q, K, V, G, s, schedule=sched)
        assert torch.equal(s.output.values, ref.output.values)
        for a, b in ((g.dq, ref_g.dq), (g.dk, ref_g.dk), (g.dv, ref_g.dv)):
            assert torch.equal(a.values, b.values)
