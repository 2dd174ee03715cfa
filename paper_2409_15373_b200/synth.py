"""Synthetic-input generators with the reference's pinned algorithms (harness, not compute).

The reference's generator (rng.hpp:10-28, rng.cpp:35-64) is std::mt19937_64 with modulo-method
bounded integers and 53-bit reals; lengths come from gen_lengths (fixed / uniform / half-mean).
Configs 2 and 5 use the Zipf generator SURVEY.md §8(d) defines. Reproducing them bit-exactly here
lets bench.py build exactly the BASELINE workloads without touching oracle/ (tests/test_synth.py pins
this module against the oracle and the compiled reference).
"""
from __future__ import annotations

import numpy as np

_N, _M = 312, 156
_UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
_MASK = (1 << 64) - 1


class Rng:
    """std::mt19937_64."""

    def __init__(self, seed: int):
        mt = [seed & _MASK]
        for i in range(1, _N):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & _MASK)
        self.mt, self.idx = mt, _N

    def _twist(self):
        mt = self.mt
        for i in range(_N):
            x = (mt[i] & _UM) | (mt[(i + 1) % _N] & _LM)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + _M) % _N] ^ xa
        self.idx = 0

    def next_u64(self) -> int:
        if self.idx >= _N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK

    def uniform_int(self, lo: int, hi: int) -> int:
        span = (hi - lo + 1) & _MASK
        if span == 0:
            return self.next_u64()
        return lo + self.next_u64() % span

    def uniform_real(self, lo: float, hi: float) -> float:
        return lo + float(self.next_u64() >> 11) * (2.0 ** -53) * (hi - lo)


def gen_lengths(kind: str, max_len: int, seed: int, batch: int, alpha: float = 1.1) -> np.ndarray:
    """rng.cpp:35-57 (fixed / uniform / half-mean) plus Zipf."""
    if batch < 1:
        raise ValueError("gen_lengths: batch must be >= 1")
    if max_len < 1:
        raise ValueError("gen_lengths: max_len must be >= 1")
    r = Rng(seed)
    out = np.empty(batch, np.int64)
    if kind == "fixed":
        out[:] = max_len
    elif kind == "uniform":
        for i in range(batch):
            out[i] = r.uniform_int(1, max_len)
    elif kind in ("half-mean", "half_mean"):
        for i in range(0, batch - 1, 2):
            u = r.uniform_int(0, max_len)
            out[i], out[i + 1] = u, max_len - u
        if batch % 2 == 1:
            out[batch - 1] = r.uniform_int(0, max_len)
    elif kind == "zipf":
        w = np.power(np.arange(1, max_len + 1, dtype=np.float64), -alpha)
        cdf = np.cumsum(w)
        cdf = cdf / cdf[-1]
        cdf[-1] = 1.0
        u = np.array([r.uniform_real(0.0, 1.0) for _ in range(batch)])
        out[:] = np.searchsorted(cdf, u, side="left") + 1
    else:
        raise ValueError(f"unknown length distribution: {kind}")
    return out


def offsets_of(lengths) -> np.ndarray:
    ln = np.asarray(lengths, np.int64)
    return np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
