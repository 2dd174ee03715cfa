"""Generates tests/golden/*.npz from THE REFERENCE ITSELF (oracle/_ref/libjagged_ref.so).

Run in the build container (where /root/reference exists and `make -C oracle` has built the
reference from its own sources):  python tests/golden/make_golden.py
The fixtures are committed; the GPU box only reads them.

Contents
  kat.npz        SPEC.md known-answer vectors as computed by the
                 reference, plus the literal expected values from the spec.
  ops.npz        every Table-1 operator and VJP on lengths {0,1,2,5,7,17,33,70}, D=16, T=8 with
                 inputs drawn by the reference's own Rng(seed+1) in bench order (bench.cpp:188-202).
  attention.npz  jagged_attention (unfused) + jagged_flash_attention fwd/bwd at blocks (3,3) and
                 (64,64) on lengths {0,1,2,5,7,17,33,70,130,257}, D=16, binary64 (attention.cpp:162-289).
  lengths.npz    gen_lengths outputs for the BASELINE configs (rng.cpp:35-57), for bit-exact checks.
  next.npz       SURVEY §8f-1 feature_interaction (attention.cpp:291-309; f64 and f32), §8f-4
                 dense_flash_attention (attention.cpp:106-160; f64 blocks (3,4)/(64,64) and f32) and §8f-2
                 jagged_mlp forward (f64, f32) + VJP (f64) (linalg.cpp:265-277, :509-573).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import reference as F  # noqa: E402


def main() -> None:
    # ---------------------------------------------------------------- KATs
    kat = {}
    off = F.make_offsets([2, 1])
    x = np.array([[1, 2], [3, 4], [5, 6]], np.float64)
    w = np.array([[[1], [1]], [[2], [0]]], np.float64)
    kat["jdbmm_out"] = F.jagged_dense_bmm(off, x, w).reshape(-1)
    kat["jdbmm_expect"] = np.array([3.0, 7.0, 10.0])
    off1 = F.make_offsets([2])
    kat["jjbmm_out"] = F.jagged_jagged_bmm(off1, np.eye(2), np.array([[2.0], [3.0]])).reshape(-1)
    kat["jjbmm_expect"] = np.array([2.0, 3.0])
    kat["jsoftmax_out"] = F.jagged_softmax(off1, np.array([[0.0], [np.log(2.0)]])).reshape(-1)
    kat["jsoftmax_expect"] = np.array([1 / 3, 2 / 3])
    kat["j2softmax_out"] = F.jagged2_softmax(off1, np.array([0.0, np.log(3.0), 0.0, 0.0]))
    kat["j2softmax_expect"] = np.array([0.25, 0.75, 0.5, 0.5])
    one = F.make_offsets([1])
    kat["jsoftmax_single"] = F.jagged_softmax(one, np.array([[123.0, -7.0]])).reshape(-1)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kat)

    # ---------------------------------------------------------------- operators + VJPs
    lens = np.array([0, 1, 2, 5, 7, 17, 33, 70], np.int64)
    off = F.make_offsets(lens)
    B, D, T, S = len(lens), 16, 8, int(off[-1])
    SQ = int((lens * lens).sum())
    seed = 42
    vals = F.uniform_values(seed + 1, 10 * S * D + 4 * SQ + 4 * B * D * T)
    cur = [0]

    def take(n, shape):
        a = vals[cur[0]:cur[0] + n].reshape(shape)
        cur[0] += n
        return a

    o = dict(offsets=off, D=D, T=T)
    o["x"] = take(S * D, (S, D))
    o["w"] = take(B * D * T, (B, D, T))
    o["y"] = take(S * T, (S, T))
    o["k"] = take(S * D, (S, D))
    o["a"] = take(SQ, (SQ,))
    o["go_t"] = take(S * T, (S, T))
    o["go_d"] = take(S * D, (S, D))
    o["go_dt"] = take(B * D * T, (B, D, T))
    o["go_sq"] = take(SQ, (SQ,))
    o["jagged_dense_bmm"] = F.jagged_dense_bmm(off, o["x"], o["w"])
    o["jagged_jagged_bmm"] = F.jagged_jagged_bmm(off, o["x"], o["y"])
    o["jagged_softmax"] = F.jagged_softmax(off, o["x"])
    o["jagged_jagged_bmm_jagged_out"] = F.jagged_jagged_bmm_jagged_out(off, o["x"], o["k"])
    o["array_jagged_bmm_jagged_out"] = F.array_jagged_bmm_jagged_out(off, o["a"], o["x"])
    o["jagged2_softmax"] = F.jagged2_softmax(off, o["a"])
    o["jagged_dense_bmm_vjp_dx"], o["jagged_dense_bmm_vjp_dw"] = F.jagged_dense_bmm_vjp(off, o["x"], o["w"], o["go_t"])
    o["jagged_jagged_bmm_vjp_dx"], o["jagged_jagged_bmm_vjp_dy"] = F.jagged_jagged_bmm_vjp(off, o["x"], o["y"], o["go_dt"])
    o["jagged_softmax_vjp"] = F.jagged_softmax_vjp(off, o["x"], o["go_d"])
    o["jjbmm_jout_vjp_dq"], o["jjbmm_jout_vjp_dk"] = F.jagged_jagged_bmm_jagged_out_vjp(off, o["x"], o["k"], o["go_sq"])
    o["ajbmm_jout_vjp_da"], o["ajbmm_jout_vjp_dv"] = F.array_jagged_bmm_jagged_out_vjp(off, o["a"], o["x"], o["go_d"])
    o["jagged2_softmax_vjp"] = F.jagged2_softmax_vjp(off, o["a"], o["go_sq"])
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **o)

    # ---------------------------------------------------------------- attention
    lens = np.array([0, 1, 2, 5, 7, 17, 33, 70, 130, 257], np.int64)
    off = F.make_offsets(lens)
    S, D = int(off[-1]), 16
    vals = F.uniform_values(7 + 1, 4 * S * D)
    q, k, v, go = (vals[i * S * D:(i + 1) * S * D].reshape(S, D) for i in range(4))
    at = dict(offsets=off, q=q, k=k, v=v, go=go)
    at["jagged_attention"] = F.jagged_attention(off, q, k, v)
    for bq, bk in [(3, 3), (64, 64)]:
        out, lse = F.jfa_forward(off, q, k, v, bq, bk)
        dq, dk, dv = F.jfa_backward(off, q, k, v, go, out, lse, bq, bk)
        tag = f"b{bq}x{bk}"
        at[f"out_{tag}"], at[f"lse_{tag}"] = out, lse
        at[f"dq_{tag}"], at[f"dk_{tag}"], at[f"dv_{tag}"] = dq, dk, dv
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **at)

    # ---------------------------------------------------------------- BASELINE length configs
    ln = {}
    ln["cfg1_uniform_B64_L128"] = F.gen_lengths("uniform", 128, 0, 64)
    ln["cfg3_halfmean_B1024_L1024"] = F.gen_lengths("half-mean", 1024, 0, 1024)
    ln["cfg4_halfmean_B2048_L1024"] = F.gen_lengths("half-mean", 1024, 0, 2048)
    ln["uniform_B33_L50_s9"] = F.gen_lengths("uniform", 50, 9, 33)
    ln["halfmean_B33_L50_s9"] = F.gen_lengths("half-mean", 50, 9, 33)
    np.savez_compressed(os.path.join(HERE, "lengths.npz"), **ln)

    # ---------------------------------------------------------------- §8f next rows
    nx = {}
    lens = np.array([0, 1, 2, 5, 7, 17, 33, 70], np.int64)
    off = F.make_offsets(lens)
    S, D, Tq = int(off[-1]), 16, 3
    vals = F.uniform_values(11, 2 * S * D + len(lens) * Tq * D)
    kf, vf = vals[:S * D].reshape(S, D), vals[S * D:2 * S * D].reshape(S, D)
    tg = vals[2 * S * D:].reshape(len(lens), Tq, D)
    nx["fi_off"], nx["fi_k"], nx["fi_v"], nx["fi_targets"] = off, kf, vf, tg
    nx["fi_out_f64"] = F.feature_interaction(off, kf, vf, tg)
    nx["fi_out_f32"] = F.feature_interaction(off, kf.astype(np.float32), vf.astype(np.float32),
                                             tg.astype(np.float32), prec="f32")
    rows, dims = 37, [16, 24, 8]
    mv = F.uniform_values(12, rows * dims[0] + dims[0] * dims[1] + dims[1] + dims[1] * dims[2] + dims[2] + rows * dims[2])
    c = 0

    def take(n):
        nonlocal c
        c += n
        return mv[c - n:c]

    x = take(rows * dims[0]).reshape(rows, dims[0])
    w0, b0 = take(dims[0] * dims[1]).reshape(dims[0], dims[1]), take(dims[1])
    w1, b1 = take(dims[1] * dims[2]).reshape(dims[1], dims[2]), take(dims[2])
    go = take(rows * dims[2]).reshape(rows, dims[2])
    layers = [(w0, b0, True), (w1, b1, False)]
    nx["mlp_x"], nx["mlp_w0"], nx["mlp_b0"], nx["mlp_w1"], nx["mlp_b1"], nx["mlp_go"] = x, w0, b0, w1, b1, go
    nx["mlp_out_f64"] = F.jagged_mlp(x, layers)
    nx["mlp_out_f32"] = F.jagged_mlp(x.astype(np.float32), [(w.astype(np.float32), b.astype(np.float32), r)
                                                            for w, b, r in layers], prec="f32")
    dx, g = F.jagged_mlp_vjp(x, layers, go)
    nx["mlp_dx"], nx["mlp_dw0"], nx["mlp_db0"], nx["mlp_dw1"], nx["mlp_db1"] = dx, g[0][0], g[0][1], g[1][0], g[1][1]
    # §8f-4: the reference's padded dense_flash_attention (attention.cpp:106-160), f64 and f32, with
    # lengths 0 (fully masked sample), L, and partial; blocks (3, 4) and (64, 64)
    dl = np.array([5, 0, 9, 3, 1], np.int64)
    Bd, Ld, Dd = len(dl), 9, 8
    dv = F.uniform_values(41, 3 * Bd * Ld * Dd)
    dq_, dk_, dv_ = (dv[i * Bd * Ld * Dd:(i + 1) * Bd * Ld * Dd].reshape(Bd, Ld, Dd) for i in range(3))
    nx["df_len"], nx["df_q"], nx["df_k"], nx["df_v"] = dl, dq_, dk_, dv_
    for bq, bk in ((3, 4), (64, 64)):
        nx[f"df_out_f64_{bq}_{bk}"], nx[f"df_lse_f64_{bq}_{bk}"] = F.dense_flash_attention(dl, dq_, dk_, dv_, bq, bk)
    nx["df_out_f32"], nx["df_lse_f32"] = F.dense_flash_attention(dl, dq_.astype(np.float32), dk_.astype(np.float32),
                                                                 dv_.astype(np.float32), 64, 64, prec="f32")
    np.savez_compressed(os.path.join(HERE, "next.npz"), **nx)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
