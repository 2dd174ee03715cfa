"""numpy/ctypes front end of oracle/jagged_oracle.c (TEST INFRASTRUCTURE ONLY).

Every function returns float64 numpy arrays computed by the C restatement, which follows the
reference loop nests cited in jagged_oracle.c. Inputs are converted to float64 first (the f64
oracle instantiation the parity tests compare against).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_I64 = C.c_int64


def build() -> None:
    """Compile liboracle.so (and, where /root/reference exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        sig = {
            "or_gen_lengths": [C.c_int, _I64, C.c_uint64, _I64, C.c_double, _i64p],
            "or_make_offsets": [_i64p, _I64, _i64p],
            "or_sq_offsets": [_i64p, _I64, _i64p],
            "or_jagged_to_dense": [_i64p, _I64, _I64, _f64p, _I64, C.c_double, _f64p],
            "or_dense_to_jagged": [_f64p, _I64, _I64, _I64, _i64p, _f64p],
            "or_jagged2_to_dense": [_i64p, _I64, _f64p, _I64, C.c_double, _f64p],
            "or_dense_to_jagged2": [_f64p, _I64, _I64, _i64p, _f64p],
            "or_jagged_dense_bmm": [_i64p, _I64, _I64, _I64, _f64p, _f64p, _f64p],
            "or_jagged_jagged_bmm": [_i64p, _I64, _I64, _I64, _f64p, _f64p, _f64p],
            "or_jagged_softmax": [_i64p, _I64, _I64, _f64p, _f64p],
            "or_jagged_jagged_bmm_jagged_out": [_i64p, _I64, _I64, _f64p, _f64p, _f64p],
            "or_array_jagged_bmm_jagged_out": [_i64p, _I64, _I64, _f64p, _f64p, _f64p],
            "or_jagged2_softmax": [_i64p, _I64, _f64p, _f64p],
            "or_jagged_dense_bmm_vjp": [_i64p, _I64, _I64, _I64, _f64p, _f64p, _f64p, _f64p, _f64p],
            "or_jagged_jagged_bmm_vjp": [_i64p, _I64, _I64, _I64, _f64p, _f64p, _f64p, _f64p, _f64p],
            "or_jagged_softmax_vjp": [_i64p, _I64, _I64, _f64p, _f64p, _f64p],
            "or_jagged_jagged_bmm_jagged_out_vjp": [_i64p, _I64, _I64, _f64p, _f64p, _f64p, _f64p, _f64p],
            "or_array_jagged_bmm_jagged_out_vjp": [_i64p, _I64, _I64, _f64p, _f64p, _f64p, _f64p, _f64p],
            "or_jagged2_softmax_vjp": [_i64p, _I64, _f64p, _f64p, _f64p],
            "or_jagged_attention": [_i64p, _I64, _I64, _f64p, _f64p, _f64p, _f64p],
            "or_jfa_forward": [_i64p, _I64, _I64, _f64p, _f64p, _f64p, _I64, _I64, _f64p, _f64p],
            "or_jfa_backward": [_i64p, _I64, _I64, _f64p, _f64p, _f64p, _f64p, _f64p, _f64p, _I64,
                                _f64p, _f64p, _f64p],
            "or_dense_attention": [_i64p, _I64, _I64, _I64, _f64p, _f64p, _f64p, _f64p],
            "or_dense_flash_attention": [_i64p, _I64, _I64, _I64, _I64, _I64, _f64p, _f64p, _f64p, _f64p, _f64p],
            "or_feature_interaction": [_i64p, _I64, _I64, _I64, _f64p, _f64p, _f64p, C.c_int, _f64p],
            "or_jagged_mlp": [_I64, C.c_int, _i64p, _f64p, _f64p, C.POINTER(C.c_int), _f64p, _f64p],
            "or_jagged_mlp_vjp": [_I64, C.c_int, _i64p, _f64p, _f64p, C.POINTER(C.c_int), _f64p, _f64p,
                                  _f64p, _f64p, _f64p],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.or_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.or_rng_seed.restype = None
        L.or_uniform_values.argtypes = [C.c_void_p, _I64, C.c_double, C.c_double, C.c_int, _f64p]
        L.or_uniform_values.restype = None
        L.or_rng_next.argtypes = [C.c_void_p]
        L.or_rng_next.restype = C.c_uint64
        L.or_sum_sq.argtypes = [_i64p, _I64]
        L.or_sum_sq.restype = C.c_int64
        _lib = L
    return _lib


class OracleError(ValueError):
    pass


def _chk(rc: int) -> None:
    if rc != 0:
        raise OracleError(lib().or_last_error().decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


# ------------------------------------------------------------------ RNG / synthetic inputs
KINDS = {"fixed": 0, "uniform": 1, "half-mean": 2, "half_mean": 2, "zipf": 3}


class Rng:
    """std::mt19937_64-based generator restated in C (rng.hpp:14-28)."""

    _SIZE = 312 * 8 + 16

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(self._SIZE)
        lib().or_rng_seed(self._buf, C.c_uint64(seed))

    def next_u64(self) -> int:
        return int(lib().or_rng_next(self._buf))

    def uniform_values(self, n: int, lo: float = -1.0, hi: float = 1.0, as_float: bool = True):
        out = np.empty(int(n), np.float64)
        if n:
            lib().or_uniform_values(self._buf, int(n), lo, hi, 1 if as_float else 0, out)
        return out


def gen_lengths(kind: str, max_len: int, seed: int, batch: int, alpha: float = 1.1) -> np.ndarray:
    out = np.empty(int(batch), np.int64)
    _chk(lib().or_gen_lengths(KINDS[kind], int(max_len), C.c_uint64(seed), int(batch), float(alpha), out))
    return out


def make_offsets(lengths) -> np.ndarray:
    lengths = _i64(lengths)
    off = np.empty(len(lengths) + 1, np.int64)
    _chk(lib().or_make_offsets(lengths, len(lengths), off))
    return off


def sq_offsets(off) -> np.ndarray:
    off = _i64(off)
    sq = np.empty(len(off), np.int64)
    _chk(lib().or_sq_offsets(off, len(off) - 1, sq))
    return sq


def sum_sq(off) -> int:
    off = _i64(off)
    return int(lib().or_sum_sq(off, len(off) - 1))


# ------------------------------------------------------------------ layout conversions
def jagged_to_dense(off, x, max_len, pad=0.0):
    off, x = _i64(off), _f64(x)
    B, D = len(off) - 1, x.shape[1]
    out = np.empty((B, max_len, D), np.float64)
    _chk(lib().or_jagged_to_dense(off, B, D, x.reshape(-1), max_len, pad, out.reshape(-1)))
    return out


def dense_to_jagged(d, lengths):
    d, lengths = _f64(d), _i64(lengths)
    B, L, D = d.shape
    out = np.empty((int(max(lengths.clip(0).sum(), 0)), D), np.float64)
    _chk(lib().or_dense_to_jagged(d.reshape(-1), B, L, D, lengths, out.reshape(-1)))
    return out


def jagged2_to_dense(off, s, max_len, pad=0.0):
    off, s = _i64(off), _f64(s)
    B = len(off) - 1
    out = np.empty((B, max_len, max_len), np.float64)
    _chk(lib().or_jagged2_to_dense(off, B, s, max_len, pad, out.reshape(-1)))
    return out


def dense_to_jagged2(d, lengths):
    d, lengths = _f64(d), _i64(lengths)
    B, L, _ = d.shape
    out = np.empty(int((lengths.clip(0) ** 2).sum()), np.float64)
    _chk(lib().or_dense_to_jagged2(d.reshape(-1), B, L, lengths, out))
    return out


# ------------------------------------------------------------------ operators
def jagged_dense_bmm(off, x, w):
    off, x, w = _i64(off), _f64(x), _f64(w)
    B, D, T = w.shape
    out = np.empty((x.shape[0], T), np.float64)
    _chk(lib().or_jagged_dense_bmm(off, B, D, T, x.reshape(-1), w.reshape(-1), out.reshape(-1)))
    return out


def jagged_jagged_bmm(off, x, y):
    off, x, y = _i64(off), _f64(x), _f64(y)
    B, D, T = len(off) - 1, x.shape[1], y.shape[1]
    out = np.empty((B, D, T), np.float64)
    _chk(lib().or_jagged_jagged_bmm(off, B, D, T, x.reshape(-1), y.reshape(-1), out.reshape(-1)))
    return out


def jagged_softmax(off, x):
    off, x = _i64(off), _f64(x)
    out = np.zeros_like(x)
    _chk(lib().or_jagged_softmax(off, len(off) - 1, x.shape[1], x.reshape(-1), out.reshape(-1)))
    return out


def jagged_jagged_bmm_jagged_out(off, q, k):
    off, q, k = _i64(off), _f64(q), _f64(k)
    out = np.empty(sum_sq(off), np.float64)
    _chk(lib().or_jagged_jagged_bmm_jagged_out(off, len(off) - 1, q.shape[1], q.reshape(-1), k.reshape(-1), out))
    return out


def array_jagged_bmm_jagged_out(off, a, v):
    off, a, v = _i64(off), _f64(a), _f64(v)
    out = np.empty_like(v)
    _chk(lib().or_array_jagged_bmm_jagged_out(off, len(off) - 1, v.shape[1], a, v.reshape(-1), out.reshape(-1)))
    return out


def jagged2_softmax(off, s):
    off, s = _i64(off), _f64(s)
    out = np.empty_like(s)
    _chk(lib().or_jagged2_softmax(off, len(off) - 1, s, out))
    return out


def jagged_dense_bmm_vjp(off, x, w, go):
    off, x, w, go = _i64(off), _f64(x), _f64(w), _f64(go)
    B, D, T = w.shape
    dx, dw = np.empty_like(x), np.empty_like(w)
    _chk(lib().or_jagged_dense_bmm_vjp(off, B, D, T, x.reshape(-1), w.reshape(-1), go.reshape(-1),
                                       dx.reshape(-1), dw.reshape(-1)))
    return dx, dw


def jagged_jagged_bmm_vjp(off, x, y, go):
    off, x, y, go = _i64(off), _f64(x), _f64(y), _f64(go)
    B, D, T = go.shape
    dx, dy = np.empty_like(x), np.empty_like(y)
    _chk(lib().or_jagged_jagged_bmm_vjp(off, B, D, T, x.reshape(-1), y.reshape(-1), go.reshape(-1),
                                        dx.reshape(-1), dy.reshape(-1)))
    return dx, dy


def jagged_softmax_vjp(off, x, go):
    off, x, go = _i64(off), _f64(x), _f64(go)
    dx = np.zeros_like(x)
    _chk(lib().or_jagged_softmax_vjp(off, len(off) - 1, x.shape[1], x.reshape(-1), go.reshape(-1), dx.reshape(-1)))
    return dx


def jagged_jagged_bmm_jagged_out_vjp(off, q, k, go):
    off, q, k, go = _i64(off), _f64(q), _f64(k), _f64(go)
    dq, dk = np.empty_like(q), np.empty_like(k)
    _chk(lib().or_jagged_jagged_bmm_jagged_out_vjp(off, len(off) - 1, q.shape[1], q.reshape(-1), k.reshape(-1),
                                                   go, dq.reshape(-1), dk.reshape(-1)))
    return dq, dk


def array_jagged_bmm_jagged_out_vjp(off, a, v, go):
    off, a, v, go = _i64(off), _f64(a), _f64(v), _f64(go)
    da, dv = np.empty_like(a), np.empty_like(v)
    _chk(lib().or_array_jagged_bmm_jagged_out_vjp(off, len(off) - 1, v.shape[1], a, v.reshape(-1),
                                                  go.reshape(-1), da, dv.reshape(-1)))
    return da, dv


def jagged2_softmax_vjp(off, s, go):
    off, s, go = _i64(off), _f64(s), _f64(go)
    ds = np.empty_like(s)
    _chk(lib().or_jagged2_softmax_vjp(off, len(off) - 1, s, go, ds))
    return ds


def jagged_attention(off, q, k, v):
    off, q, k, v = _i64(off), _f64(q), _f64(k), _f64(v)
    out = np.zeros_like(q)
    _chk(lib().or_jagged_attention(off, len(off) - 1, q.shape[1], q.reshape(-1), k.reshape(-1),
                                   v.reshape(-1), out.reshape(-1)))
    return out


def jfa_forward(off, q, k, v, block_q=64, block_k=64):
    off, q, k, v = _i64(off), _f64(q), _f64(k), _f64(v)
    out = np.empty_like(q)
    lse = np.empty(q.shape[0], np.float64)
    _chk(lib().or_jfa_forward(off, len(off) - 1, q.shape[1], q.reshape(-1), k.reshape(-1), v.reshape(-1),
                              block_q, block_k, out.reshape(-1), lse))
    return out, lse


def jfa_backward(off, q, k, v, go, out, lse, block_k=64):
    off = _i64(off)
    q, k, v, go, out, lse = map(_f64, (q, k, v, go, out, lse))
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    _chk(lib().or_jfa_backward(off, len(off) - 1, q.shape[1], q.reshape(-1), k.reshape(-1), v.reshape(-1),
                               go.reshape(-1), out.reshape(-1), lse, block_k, dq.reshape(-1),
                               dk.reshape(-1), dv.reshape(-1)))
    return dq, dk, dv


def dense_attention(lengths, q, k, v):
    lengths = _i64(lengths)
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, L, D = q.shape
    out = np.empty_like(q)
    _chk(lib().or_dense_attention(lengths, B, L, D, q.reshape(-1), k.reshape(-1), v.reshape(-1), out.reshape(-1)))
    return out


def dense_flash_attention(lengths, q, k, v, block_q=64, block_k=64):
    """attention.cpp:106-160 -> (out [B, L, D], lse [B*L]) (jagged_oracle.c or_dense_flash_attention)."""
    lengths = _i64(lengths)
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, L, D = q.shape
    out = np.empty_like(q)
    lse = np.empty(B * L)
    _chk(lib().or_dense_flash_attention(lengths, B, L, D, block_q, block_k, q.reshape(-1), k.reshape(-1),
                                        v.reshape(-1), out.reshape(-1), lse))
    return out, lse


def feature_interaction(off, k_feat, v_feat, targets, as_float=False):
    """attention.cpp:291-309 -> [B, Tq, D] (jagged_oracle.c or_feature_interaction)."""
    off, k_feat, v_feat, targets = _i64(off), _f64(k_feat), _f64(v_feat), _f64(targets)
    B, Tq, D = targets.shape
    out = np.zeros((B, Tq, D), np.float64)
    _chk(lib().or_feature_interaction(off, B, D, Tq, k_feat.reshape(-1), v_feat.reshape(-1), targets.reshape(-1),
                                      1 if as_float else 0, out.reshape(-1)))
    return out


def _mlp_pack(layers):
    """layers: [(W [d_in, d_out], b [d_out], relu bool)] -> (dims, w, b, relu) flat arrays."""
    dims = np.array([layers[0][0].shape[0]] + [w.shape[1] for w, _, _ in layers], np.int64)
    w = np.concatenate([_f64(w).reshape(-1) for w, _, _ in layers])
    b = np.concatenate([_f64(b).reshape(-1) for _, b, _ in layers])
    relu = (C.c_int * len(layers))(*[1 if r else 0 for _, _, r in layers])
    return dims, w, b, relu


def jagged_mlp(x, layers):
    """linalg.cpp:265-277 (activations in binary64 between layers)."""
    x = _f64(x)
    dims, w, b, relu = _mlp_pack(layers)
    out = np.empty((x.shape[0], int(dims[-1])), np.float64)
    _chk(lib().or_jagged_mlp(x.shape[0], len(layers), dims, w, b, relu, x.reshape(-1), out.reshape(-1)))
    return out


def jagged_mlp_vjp(x, layers, go):
    """linalg.cpp:509-573 -> (dx, [(dW, db) per layer])."""
    x, go = _f64(x), _f64(go)
    dims, w, b, relu = _mlp_pack(layers)
    dx = np.empty_like(x)
    dw, db = np.empty_like(w), np.empty_like(b)
    _chk(lib().or_jagged_mlp_vjp(x.shape[0], len(layers), dims, w, b, relu, x.reshape(-1), go.reshape(-1),
                                 dx.reshape(-1), dw, db))
    grads, wo, bo = [], 0, 0
    for l in range(len(layers)):
        di, do = int(dims[l]), int(dims[l + 1])
        grads.append((dw[wo:wo + di * do].reshape(di, do), db[bo:bo + do].copy()))
        wo, bo = wo + di * do, bo + do
    return dx, grads
