"""ctypes front end of oracle/_ref/libjagged_ref.so — the REFERENCE ITSELF (test infrastructure).

The .so is compiled by oracle/Makefile from the reference's own sources under /root/reference
(never copied into the repo) plus oracle/ref_shim.cpp. It travels to the GPU box inside the repo
snapshot (oracle/_ref is git-ignored but not gpurun-ignored). Used to pin oracle/jagged_oracle.c,
to generate tests/golden fixtures and to time the reference CPU path in bench.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libjagged_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_hardware_threads.restype = C.c_int
    return _lib


class ReferenceError(ValueError):
    pass


def _chk(rc):
    if rc != 0:
        raise ReferenceError(lib().ref_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _arr(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=dt))


_DT = {"f32": np.float32, "f64": np.float64}
_I = C.c_int64


def hardware_threads() -> int:
    return int(lib().ref_hardware_threads())


def gen_lengths(kind: str, max_len: int, seed: int, batch: int) -> np.ndarray:
    k = {"fixed": 0, "uniform": 1, "half-mean": 2, "half_mean": 2}[kind]
    out = np.empty(batch, np.int64)
    _chk(lib().ref_gen_lengths(C.c_int(k), _I(max_len), C.c_uint64(seed), _I(batch), _p(out)))
    return out


def uniform_values(seed: int, n: int, lo=-1.0, hi=1.0, prec="f64") -> np.ndarray:
    out = np.empty(n, _DT[prec])
    fn = lib().ref_uniform_values_f64 if prec == "f64" else lib().ref_uniform_values_f32
    _chk(fn(C.c_uint64(seed), _I(n), C.c_double(lo), C.c_double(hi), _p(out)))
    return out


class RngStream:
    """One jagged::Rng(seed) stream; successive uniform_f32 calls continue it (bench.cpp:323-329 draws q, k, v
    and then grad_out from Rng(seed + 1) in that order)."""

    def __init__(self, seed: int):
        lib().ref_rng_new.restype = C.c_void_p
        self._h = C.c_void_p(lib().ref_rng_new(C.c_uint64(seed)))

    def uniform_f32(self, n: int, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(int(n), np.float32)
        _chk(lib().ref_rng_uniform_f32(self._h, _I(int(n)), C.c_double(lo), C.c_double(hi), _p(out)))
        return out

    def __del__(self):
        try:
            lib().ref_rng_free(self._h)
        except Exception:
            pass


def set_vjp_threads(threads: int) -> None:
    """KernelOptions.threads for the reference VJPs (default 1, as the reference registry calls them)."""
    lib().ref_set_vjp_threads(C.c_int(int(threads)))


def make_offsets(lengths) -> np.ndarray:
    lengths = _arr(lengths, np.int64)
    off = np.empty(len(lengths) + 1, np.int64)
    _chk(lib().ref_make_offsets(_p(lengths), _I(len(lengths)), _p(off)))
    return off


def jagged_to_dense(off, x, L, pad=0.0):
    off, x = _arr(off, np.int64), _arr(x, np.float64)
    B, D = len(off) - 1, x.shape[1]
    out = np.empty((B, L, D), np.float64)
    _chk(lib().ref_jagged_to_dense_f64(_p(off), _I(B), _I(D), _p(x), _I(L), C.c_double(pad), _p(out)))
    return out


def _sumsq(off):
    ln = np.diff(off)
    return int((ln * ln).sum())


def jagged_dense_bmm(off, x, w, prec="f64", threads=1):
    dt = _DT[prec]
    off, x, w = _arr(off, np.int64), _arr(x, dt), _arr(w, dt)
    B, D, T = w.shape
    out = np.empty((x.shape[0], T), dt)
    _chk(getattr(lib(), f"ref_jagged_dense_bmm_{prec}")(_p(off), _I(B), _I(D), _I(T), _p(x), _p(w), threads, _p(out)))
    return out


def jagged_jagged_bmm(off, x, y, prec="f64", threads=1):
    dt = _DT[prec]
    off, x, y = _arr(off, np.int64), _arr(x, dt), _arr(y, dt)
    B, D, T = len(off) - 1, x.shape[1], y.shape[1]
    out = np.empty((B, D, T), dt)
    _chk(getattr(lib(), f"ref_jagged_jagged_bmm_{prec}")(_p(off), _I(B), _I(D), _I(T), _p(x), _p(y), threads, _p(out)))
    return out


def jagged_softmax(off, x, prec="f64", threads=1):
    dt = _DT[prec]
    off, x = _arr(off, np.int64), _arr(x, dt)
    out = np.empty_like(x)
    _chk(getattr(lib(), f"ref_jagged_softmax_{prec}")(_p(off), _I(len(off) - 1), _I(x.shape[1]), _p(x), threads, _p(out)))
    return out


def jagged_jagged_bmm_jagged_out(off, q, k, prec="f64", threads=1):
    dt = _DT[prec]
    off, q, k = _arr(off, np.int64), _arr(q, dt), _arr(k, dt)
    out = np.empty(_sumsq(off), dt)
    _chk(getattr(lib(), f"ref_jagged_jagged_bmm_jagged_out_{prec}")(_p(off), _I(len(off) - 1), _I(q.shape[1]),
                                                                    _p(q), _p(k), threads, _p(out)))
    return out


def array_jagged_bmm_jagged_out(off, a, v, prec="f64", threads=1):
    dt = _DT[prec]
    off, a, v = _arr(off, np.int64), _arr(a, dt), _arr(v, dt)
    out = np.empty_like(v)
    _chk(getattr(lib(), f"ref_array_jagged_bmm_jagged_out_{prec}")(_p(off), _I(len(off) - 1), _I(v.shape[1]),
                                                                   _p(a), _p(v), threads, _p(out)))
    return out


def jagged2_softmax(off, s, prec="f64", threads=1):
    dt = _DT[prec]
    off, s = _arr(off, np.int64), _arr(s, dt)
    out = np.empty_like(s)
    _chk(getattr(lib(), f"ref_jagged2_softmax_{prec}")(_p(off), _I(len(off) - 1), _p(s), threads, _p(out)))
    return out


def jagged_attention(off, q, k, v, prec="f64", threads=1):
    dt = _DT[prec]
    off = _arr(off, np.int64)
    q, k, v = (_arr(a, dt) for a in (q, k, v))
    out = np.empty_like(q)
    _chk(getattr(lib(), f"ref_jagged_attention_{prec}")(_p(off), _I(len(off) - 1), _I(q.shape[1]), _p(q), _p(k),
                                                        _p(v), threads, _p(out)))
    return out


def jfa_forward(off, q, k, v, block_q=64, block_k=64, prec="f64", threads=1):
    dt = _DT[prec]
    off = _arr(off, np.int64)
    q, k, v = (_arr(a, dt) for a in (q, k, v))
    out = np.empty_like(q)
    lse = np.empty(q.shape[0], dt)
    _chk(getattr(lib(), f"ref_jfa_forward_{prec}")(_p(off), _I(len(off) - 1), _I(q.shape[1]), _p(q), _p(k), _p(v),
                                                   _I(block_q), _I(block_k), threads, _p(out), _p(lse)))
    return out, lse


def dense_flash_attention(lengths, q, k, v, block_q=64, block_k=64, prec="f64", threads=1):
    """The reference's attention.cpp:106-160 on [B, L, D] -> (out, lse [B*L])."""
    dt = np.float64 if prec == "f64" else np.float32
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    q, k, v = (_arr(a, dt) for a in (q, k, v))
    B, L, D = q.shape
    out = np.empty_like(q)
    lse = np.empty(B * L, dt)
    _chk(getattr(lib(), f"ref_dense_flash_attention_{prec}")(_p(lengths), _I(B), _I(L), _I(D), _p(q), _p(k), _p(v),
                                                              _I(block_q), _I(block_k), threads, _p(out), _p(lse)))
    return out, lse


def jfa_backward(off, q, k, v, go, out, lse, block_q=64, block_k=64, prec="f64", threads=1):
    dt = _DT[prec]
    off = _arr(off, np.int64)
    q, k, v, go, out, lse = (_arr(a, dt) for a in (q, k, v, go, out, lse))
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    _chk(getattr(lib(), f"ref_jfa_backward_{prec}")(_p(off), _I(len(off) - 1), _I(q.shape[1]), _p(q), _p(k), _p(v),
                                                    _p(go), _p(out), _p(lse), _I(block_q), _I(block_k), threads,
                                                    _p(dq), _p(dk), _p(dv)))
    return dq, dk, dv


def _vjp2(name, off, a, b, go, outs_like, Bdims):
    off = _arr(off, np.int64)
    a, b, go = (_arr(t, np.float64) for t in (a, b, go))
    o1, o2 = (np.empty_like(t) for t in outs_like(a, b))
    _chk(getattr(lib(), name)(_p(off), *[_I(x) for x in Bdims], _p(a), _p(b), _p(go), _p(o1), _p(o2)))
    return o1, o2


def jagged_dense_bmm_vjp(off, x, w, go):
    B, D, T = np.asarray(w).shape
    return _vjp2("ref_jagged_dense_bmm_vjp_f64", off, x, w, go, lambda a, b: (a, b), (B, D, T))


def jagged_jagged_bmm_vjp(off, x, y, go):
    B, D, T = np.asarray(go).shape
    return _vjp2("ref_jagged_jagged_bmm_vjp_f64", off, x, y, go, lambda a, b: (a, b), (B, D, T))


def jagged_jagged_bmm_jagged_out_vjp(off, q, k, go):
    q = np.asarray(q)
    return _vjp2("ref_jagged_jagged_bmm_jagged_out_vjp_f64", off, q, k, go, lambda a, b: (a, b),
                 (len(off) - 1, q.shape[1]))


def array_jagged_bmm_jagged_out_vjp(off, a, v, go):
    v = np.asarray(v)
    return _vjp2("ref_array_jagged_bmm_jagged_out_vjp_f64", off, a, v, go, lambda a_, b_: (a_, b_),
                 (len(off) - 1, v.shape[1]))


def jagged_softmax_vjp(off, x, go):
    off = _arr(off, np.int64)
    x, go = _arr(x, np.float64), _arr(go, np.float64)
    dx = np.empty_like(x)
    _chk(lib().ref_jagged_softmax_vjp_f64(_p(off), _I(len(off) - 1), _I(x.shape[1]), _p(x), _p(go), _p(dx)))
    return dx


def jagged2_softmax_vjp(off, s, go):
    off = _arr(off, np.int64)
    s, go = _arr(s, np.float64), _arr(go, np.float64)
    ds = np.empty_like(s)
    _chk(lib().ref_jagged2_softmax_vjp_f64(_p(off), _I(len(off) - 1), _p(s), _p(go), _p(ds)))
    return ds


def feature_interaction(off, k_feat, v_feat, targets, prec="f64"):
    """attention.cpp:291-309 through the compiled reference."""
    dt = _DT[prec]
    off, k_feat, v_feat, targets = _arr(off, np.int64), _arr(k_feat, dt), _arr(v_feat, dt), _arr(targets, dt)
    B, Tq, D = targets.shape
    out = np.empty((B, Tq, D), dt)
    _chk(getattr(lib(), f"ref_feature_interaction_{prec}")(_p(off), _I(B), _I(D), _I(Tq), _p(k_feat), _p(v_feat),
                                                           _p(targets), _p(out)))
    return out


def _mlp_pack(layers, dt):
    dims = np.array([layers[0][0].shape[0]] + [w.shape[1] for w, _, _ in layers], np.int64)
    w = np.ascontiguousarray(np.concatenate([np.asarray(w, dt).reshape(-1) for w, _, _ in layers]))
    b = np.ascontiguousarray(np.concatenate([np.asarray(b, dt).reshape(-1) for _, b, _ in layers]))
    relu = np.array([1 if r else 0 for _, _, r in layers], np.int32)
    return dims, w, b, relu


def jagged_mlp(x, layers, prec="f64"):
    """linalg.cpp:265-277; layers = [(W [d_in, d_out], bias [d_out], relu)]."""
    dt = _DT[prec]
    x = _arr(x, dt)
    dims, w, b, relu = _mlp_pack(layers, dt)
    out = np.empty((x.shape[0], int(dims[-1])), dt)
    _chk(getattr(lib(), f"ref_jagged_mlp_{prec}")(_I(x.shape[0]), C.c_int(len(layers)), _p(dims), _p(w), _p(b),
                                                  _p(relu), _p(x), _p(out)))
    return out


def jagged_mlp_vjp(x, layers, go):
    """linalg.cpp:509-573 (binary64 instantiation, the one the reference's callers import)."""
    x, go = _arr(x, np.float64), _arr(go, np.float64)
    dims, w, b, relu = _mlp_pack(layers, np.float64)
    dx, dw, db = np.empty_like(x), np.empty_like(w), np.empty_like(b)
    _chk(lib().ref_jagged_mlp_vjp_f64(_I(x.shape[0]), C.c_int(len(layers)), _p(dims), _p(w), _p(b), _p(relu),
                                      _p(x), _p(go), _p(dx), _p(dw), _p(db)))
    grads, wo, bo = [], 0, 0
    for l in range(len(layers)):
        di, do = int(dims[l]), int(dims[l + 1])
        grads.append((dw[wo:wo + di * do].reshape(di, do), db[bo:bo + do].copy()))
        wo, bo = wo + di * do, bo + do
    return dx, grads


def cost_model(op, lengths, D, T, element_bytes=4, padded_len=None, block_q=64, block_k=64, variant=None):
    """The reference's cost_model.cpp: dict of (jagged, padded) flops/bytes/intermediate (+ variant numbers)."""
    ln = np.ascontiguousarray(lengths, dtype=np.int64)
    out = np.zeros(8, np.int64)
    _chk(lib().ref_cost_model(op.encode(), variant.encode() if variant else None, _p(ln), _I(len(ln)), _I(D), _I(T),
                              _I(element_bytes), _I(-1 if padded_len is None else padded_len), _I(block_q),
                              _I(block_k), _p(out)))
    r = {"flops": (int(out[0]), int(out[1])), "bytes": (int(out[2]), int(out[3])),
         "intermediate": (int(out[4]), int(out[5]))}
    if variant:
        r["variant"] = (int(out[6]), int(out[7]))
    return r


def csv_header() -> str:
    lib().ref_csv_header.restype = C.c_char_p
    return lib().ref_csv_header().decode()
