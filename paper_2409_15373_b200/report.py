"""Bench/report layer for the GPU variants: the reference's analytic cost model, bench records and
report renderers, so GPU timings come out in the reference's Table-1 / Figure-2 record schema.

* Cost model — restates cost_model.cpp (FLOP convention cost_model.hpp:15-27): ``flops_of`` (cost_model.cpp:101-131),
  ``intermediate_elements`` (:133-151), ``bytes_of`` (:153-193), ``variant_flops`` / ``variant_bytes``
  (:230-255). Pinned bit-exact to the compiled reference by tests/test_report.py.
* Records — ``BenchRecord`` / ``VariantStats`` mirror bench.hpp:46-77; ``render_report`` mirrors bench.cpp
  render_csv / render_json / render_md (:525-610, CSV header bench.hpp:79-81); ``parse_records_json`` is the
  inverse of the json format (bench.cpp:625-).
* ``percentile`` is the linear-interpolation percentile of bench.cpp:380-388 used for p10/p50/p90.

Timing on the device (CUDA events) and the padded torch baselines live in bench.py ``--config table1``.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

CSV_HEADER = ("op,variant,B,D,T,max_len,dist,seed,precision,threads,time_us_p50,time_us_p10,"
              "time_us_p90,flops,bytes,speedup_vs_dense,bytes_ratio_vs_dense")

_FAMILY = {
    "jagged_dense_bmm": "bmm", "jagged_jagged_bmm": "bmm",
    "jagged_jagged_bmm_jagged_out": "bmm_jagged_out", "array_jagged_bmm_jagged_out": "bmm_jagged_out",
    "jagged_softmax": "softmax", "jagged2_softmax": "softmax2", "jagged_mlp": "mlp",
    "dense_attention": "attention_naive", "jagged_attention": "attention_naive",
    "dense_flash_attention": "attention_flash", "jagged_flash_attention": "attention_flash",
}


class CostModelError(ValueError):
    pass


@dataclass
class OpConfig:
    """cost_model.hpp:29-39."""
    op_id: str
    dim: int
    t: int
    lengths: list
    element_bytes: int = 4
    padded_len: int | None = None
    block_q: int = 64
    block_k: int = 64


def _resolve(c: OpConfig):
    # cost_model.cpp:20-40
    if len(c.lengths) == 0:
        raise CostModelError("cost model: lengths required")
    if c.dim < 1 or c.t < 1 or c.element_bytes < 1:
        raise CostModelError("cost model: dim, t, element_bytes must be positive")
    ln = [int(n) for n in c.lengths]
    if any(n < 0 for n in ln):
        raise CostModelError("cost model: negative length")
    max_len = max(ln)
    if c.padded_len is not None:
        if c.padded_len < max_len:
            raise CostModelError("cost model: padded_len smaller than max length")
        max_len = int(c.padded_len)
    return ln, len(ln), sum(ln), sum(n * n for n in ln), max_len


def _family(op_id: str) -> str:
    if op_id not in _FAMILY:
        raise CostModelError(f"cost model: unknown op_id '{op_id}'")
    return _FAMILY[op_id]


def _mlp_chain(c: OpConfig):  # the benchable MLP: D -> T (relu) -> D
    return [c.dim, c.t, c.dim]


def _flash_softmax_flops(n: int, block_k: int, d: int) -> int:
    # 3 per score, 2(D+1) rescale per (row, key block), D+2 finalize per row
    if n == 0:
        return 0
    return n * (3 * n + -(-n // block_k) * 2 * (d + 1) + (d + 2))


def _attn_matmul_flops(sq: int, d: int) -> int:
    return 4 * sq * d + sq  # QK^T and PV multiply-adds + the score scaling


def flops_of(c: OpConfig) -> tuple[int, int]:
    """(jagged, padded) FLOPs."""
    ln, b, s, sq, L = _resolve(c)
    fam, d, t = _family(c.op_id), c.dim, c.t
    prow, psq = b * L, b * L * L
    if fam == "bmm":
        return 2 * s * d * t, 2 * prow * d * t
    if fam == "bmm_jagged_out":
        return 2 * sq * d, 2 * psq * d
    if fam == "softmax":
        return 4 * s * d, 4 * prow * d
    if fam == "softmax2":
        return 4 * sq, 4 * psq
    if fam == "mlp":
        ch = _mlp_chain(c)
        per_row = sum(2 * ch[i] * ch[i + 1] + 2 * ch[i + 1] for i in range(len(ch) - 1))
        return s * per_row, prow * per_row
    if fam == "attention_naive":
        return _attn_matmul_flops(sq, d) + 4 * sq, _attn_matmul_flops(psq, d) + 4 * psq
    jag = _attn_matmul_flops(sq, d) + sum(_flash_softmax_flops(n, c.block_k, d) for n in ln)
    return jag, _attn_matmul_flops(psq, d) + b * _flash_softmax_flops(L, c.block_k, d)


def intermediate_elements(c: OpConfig) -> tuple[int, int]:
    ln, b, s, sq, L = _resolve(c)
    fam = _family(c.op_id)
    if fam == "attention_naive":
        return sq, b * L * L
    if fam == "attention_flash":
        return c.block_q * c.block_k + s, c.block_q * c.block_k + b * L
    if fam == "mlp":
        hidden = max(_mlp_chain(c)[1:-1], default=0)
        return s * hidden, b * L * hidden
    return 0, 0


def bytes_of(c: OpConfig) -> tuple[int, int]:
    """(jagged, padded) bytes: element_bytes x (inputs + outputs + peak intermediate)."""
    ln, b, s, sq, L = _resolve(c)
    fam, d, t = _family(c.op_id), c.dim, c.t
    prow, psq = b * L, b * L * L
    if fam == "bmm":
        if c.op_id == "jagged_dense_bmm":
            io = (s * d + b * d * t + s * t, prow * d + b * d * t + prow * t)
        else:
            io = (s * (d + t) + b * d * t, prow * (d + t) + b * d * t)
    elif fam == "bmm_jagged_out":
        io = (2 * s * d + sq, 2 * prow * d + psq)
    elif fam == "softmax":
        io = (2 * s * d, 2 * prow * d)
    elif fam == "softmax2":
        io = (2 * sq, 2 * psq)
    elif fam == "mlp":
        ch = _mlp_chain(c)
        params = sum(ch[i] * ch[i + 1] + ch[i + 1] for i in range(len(ch) - 1))
        io = (s * (ch[0] + ch[-1]) + params, prow * (ch[0] + ch[-1]) + params)
    else:
        io = (4 * s * d, 4 * prow * d)
    sj, sp = intermediate_elements(c)
    return c.element_bytes * (io[0] + sj), c.element_bytes * (io[1] + sp)


def _variant_cfg(c: OpConfig, variant: str):
    if variant in ("jagged", "padded"):
        return c, variant == "padded"
    if variant in ("dense_attention", "dense_flash_attention"):
        return OpConfig(**{**c.__dict__, "op_id": variant}), True
    if variant in ("jagged_attention", "jagged_flash_attention"):
        return OpConfig(**{**c.__dict__, "op_id": variant}), False
    raise CostModelError(f"cost model: unknown variant '{variant}' for op '{c.op_id}'")


def variant_flops(c: OpConfig, variant: str) -> int:
    vc, padded = _variant_cfg(c, variant)
    return flops_of(vc)[1 if padded else 0]


def variant_bytes(c: OpConfig, variant: str) -> int:
    vc, padded = _variant_cfg(c, variant)
    return bytes_of(vc)[1 if padded else 0]


def cost_model_knows(op_id: str) -> bool:
    return op_id in _FAMILY


def percentile(xs, q: float) -> float:
    xs = sorted(xs)
    if not xs:
        return 0.0
    pos = q * (len(xs) - 1)
    lo = int(pos)
    hi = min(lo + 1, len(xs) - 1)
    return xs[lo] + (xs[hi] - xs[lo]) * (pos - lo)


@dataclass
class VariantStats:
    """bench.hpp:46-59 (time in microseconds; `checksum` = binary64 sum of the valid-region output)."""
    variant: str
    time_us_p50: float = 0.0
    time_us_p10: float = 0.0
    time_us_p90: float = 0.0
    flops: int = 0
    bytes: int = 0
    checksum: float = 0.0
    noisy: bool = False
    speedup_vs_dense: float = 1.0
    bytes_ratio_vs_dense: float = 1.0

    @staticmethod
    def from_times(variant: str, times_us, checksum: float = 0.0) -> "VariantStats":
        p10, p50, p90 = (percentile(times_us, q) for q in (0.1, 0.5, 0.9))
        noisy = p90 / p10 > 3.0 if p10 > 0 else p90 > 0
        return VariantStats(variant, p50, p10, p90, checksum=checksum, noisy=noisy)


@dataclass
class BenchRecord:
    """bench.hpp:61-77. `threads` is the reference's CPU thread count; GPU records carry the GPU count."""
    op_id: str
    batch: int
    dim: int
    t: int
    max_len: int
    dist: str
    seed: int
    precision: str
    threads: int = 1
    flops_jagged: int = 0
    flops_padded: int = 0
    bytes_jagged: int = 0
    bytes_padded: int = 0
    variants: list = field(default_factory=list)

    def finalize(self, cfg: OpConfig) -> "BenchRecord":
        """Fill the analytic columns and the ratios against variants[0] (the padded/dense baseline),
        bench.cpp:436-472."""
        self.flops_jagged, self.flops_padded = flops_of(cfg)
        self.bytes_jagged, self.bytes_padded = bytes_of(cfg)
        for v in self.variants:
            v.flops, v.bytes = variant_flops(cfg, v.variant), variant_bytes(cfg, v.variant)
        base = self.variants[0]
        for v in self.variants:
            v.speedup_vs_dense = base.time_us_p50 / v.time_us_p50 if v.time_us_p50 > 0 else 1.0
            v.bytes_ratio_vs_dense = v.bytes / base.bytes if base.bytes > 0 else 1.0
        return self


def _fmt_double(v: float) -> str:  # std::ostream default, precision 6
    if math.isinf(v) or math.isnan(v):
        return {True: "inf", False: "-inf"}[v > 0] if math.isinf(v) else "nan"
    return f"{v:.6g}"


def render_report(records, fmt: str) -> str:
    if not records:
        raise ValueError("render_report: no records")
    if fmt == "csv":
        rows = [CSV_HEADER]
        for r in records:
            for v in r.variants:
                rows.append(",".join([r.op_id, v.variant, str(r.batch), str(r.dim), str(r.t), str(r.max_len), r.dist,
                                      str(r.seed), r.precision, str(r.threads), f"{v.time_us_p50:.3f}",
                                      f"{v.time_us_p10:.3f}", f"{v.time_us_p90:.3f}", str(v.flops), str(v.bytes),
                                      _fmt_double(v.speedup_vs_dense), _fmt_double(v.bytes_ratio_vs_dense)]))
        return "\n".join(rows) + "\n"
    if fmt == "json":
        out = []
        for r in records:
            d = {"op": r.op_id, "B": r.batch, "D": r.dim, "T": r.t, "max_len": r.max_len, "dist": r.dist,
                 "seed": r.seed, "precision": r.precision, "threads": r.threads, "flops_jagged": r.flops_jagged,
                 "flops_padded": r.flops_padded, "bytes_jagged": r.bytes_jagged, "bytes_padded": r.bytes_padded,
                 "variants": [dict(v.__dict__) for v in r.variants]}
            out.append(d)
        return json.dumps(out, indent=2)
    if fmt == "md":
        rows = ["| op | variant | B | D | T | max_len | time_us (p50) | FLOPs (M) | memory (MB) |",
                "|---|---|---|---|---|---|---|---|---|"]
        for r in records:
            for i, v in enumerate(r.variants):
                base = i == 0 and v.speedup_vs_dense == 1.0 and v.bytes_ratio_vs_dense == 1.0
                tc, fc, bc = f"{v.time_us_p50:.1f}", f"{v.flops / 1e6:.1f}", f"{v.bytes / 1e6:.1f}"
                if not base:
                    tc += f" ({v.speedup_vs_dense:.2f}×)"
                    if v.flops > 0:
                        fc += f" ({r.flops_padded / v.flops:.2f}×)"
                    if v.bytes > 0:
                        bc += f" ({r.bytes_padded / v.bytes:.2f}×)"
                rows.append(f"| {r.op_id} | {v.variant} | {r.batch} | {r.dim} | {r.t} | {r.max_len} | {tc} | {fc} | "
                            f"{bc} |")
        return "\n".join(rows) + "\n"
    raise ValueError(f"unknown report format: {fmt}")


def parse_records_json(text: str):
    recs = []
    for d in json.loads(text):
        r = BenchRecord(d["op"], d["B"], d["D"], d["T"], d["max_len"], d["dist"], d["seed"], d["precision"],
                        d["threads"], d["flops_jagged"], d["flops_padded"], d["bytes_jagged"], d["bytes_padded"])
        r.variants = [VariantStats(**v) for v in d["variants"]]
        recs.append(r)
    return recs
