"""Parity helpers shared by the GPU tests (tolerances from BASELINE.json north_star).

fp32 mode: within 1e-5 relative of the binary64 oracle, measured norm-wise AND elementwise with an
RMS floor (|got - ref| <= tol * max(|ref|, rms(ref))) — the reference's own elementwise metric with a
1e-8 floor fails between its own f32 and f64 paths on near-zero outputs.
bf16 I/O: max-abs error <= 2e-2 against the binary64 oracle run on the same bf16-rounded inputs.
Integer/index/layout work: bit-exact.
"""
from __future__ import annotations

import numpy as np
import torch

FP32_TOL = 1e-5
BF16_MAXABS = 2e-2


def to_np(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().float().cpu().double().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().double().numpy()
    return np.asarray(t, dtype=np.float64)


def assert_fp32_close(got, ref, tol=FP32_TOL, what=""):
    g, r = to_np(got).reshape(-1), np.asarray(ref, np.float64).reshape(-1)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    if r.size == 0:
        return
    err = np.abs(g - r)
    rms = float(np.sqrt(np.mean(r * r)))
    norm_rel = float(np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-300))
    assert norm_rel <= tol, f"{what}: norm-wise rel {norm_rel:.3e} > {tol}"
    bound = tol * np.maximum(np.abs(r), rms) + 1e-30
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, (f"{what}: {bad.size} elements exceed {tol}*max(|ref|, rms); first at {bad[0]}: "
                           f"got {g[bad[0]]!r} ref {r[bad[0]]!r}")


def assert_bf16_close(got, ref, tol=BF16_MAXABS, what=""):
    g, r = to_np(got).reshape(-1), np.asarray(ref, np.float64).reshape(-1)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    if r.size == 0:
        return
    m = float(np.max(np.abs(g - r)))
    assert m <= tol, f"{what}: max-abs {m:.3e} > {tol}"


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16 and back to float64 (what the GPU sees)."""
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).double().numpy()


def f32_round(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, np.float32).astype(np.float64)
