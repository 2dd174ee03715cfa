"""the bench/report layer (paper_2409_15373_b200/report.py) against the compiled reference — the
analytic cost model bit-exact (cost_model.cpp) and the CSV schema (bench.hpp:79-81) — plus the report renderers."""
import numpy as np
import pytest

from oracle import reference as F
from paper_2409_15373_b200 import report as RP

OPS = ["jagged_dense_bmm", "jagged_jagged_bmm", "jagged_jagged_bmm_jagged_out", "array_jagged_bmm_jagged_out",
       "jagged_softmax", "jagged2_softmax", "jagged_mlp", "dense_attention", "jagged_attention",
       "dense_flash_attention", "jagged_flash_attention"]
LENGTHS = [[0, 1, 2, 5, 7, 17, 33, 70], [64, 64, 64], list(np.arange(0, 300, 37)), [1]]


@pytest.mark.skipif(not F.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("op", OPS)
def test_cost_model_matches_reference(op):
    for ln in LENGTHS:
        for D, T, eb, pl, bq, bk in ((64, 32, 4, None, 64, 64), (128, 256, 2, 400, 32, 16), (8, 8, 8, None, 3, 5)):
            variants = ["jagged", "padded"]
            if "attention" in op:
                variants += ["dense_attention", "jagged_attention", "dense_flash_attention", "jagged_flash_attention"]
            cfg = RP.OpConfig(op, D, T, ln, eb, pl, bq, bk)
            for var in variants:
                ref = F.cost_model(op, ln, D, T, eb, pl, bq, bk, variant=var)
                assert RP.flops_of(cfg) == ref["flops"], (op, ln, D, T)
                assert RP.bytes_of(cfg) == ref["bytes"], (op, ln, D, T)
                assert RP.intermediate_elements(cfg) == ref["intermediate"]
                assert (RP.variant_flops(cfg, var), RP.variant_bytes(cfg, var)) == ref["variant"], (op, var)


@pytest.mark.skipif(not F.available(), reason="oracle/_ref not built")
def test_csv_header_matches_reference():
    assert RP.CSV_HEADER == F.csv_header()


def test_cost_model_errors():
    with pytest.raises(RP.CostModelError, match="unknown op_id 'nope'"):
        RP.flops_of(RP.OpConfig("nope", 4, 4, [1]))
    with pytest.raises(RP.CostModelError, match="lengths required"):
        RP.flops_of(RP.OpConfig("jagged_softmax", 4, 4, []))
    with pytest.raises(RP.CostModelError, match="padded_len smaller than max length"):
        RP.bytes_of(RP.OpConfig("jagged_softmax", 4, 4, [5], padded_len=4))
    with pytest.raises(RP.CostModelError, match="unknown variant 'x'"):
        RP.variant_flops(RP.OpConfig("jagged_softmax", 4, 4, [5]), "x")


def _records():
    cfg = RP.OpConfig("jagged_flash_attention", 128, 1, [3, 0, 70], 2)
    rec = RP.BenchRecord("attention", 3, 128, 1, 70, "half_mean", 0, "bf16", 1)
    rec.variants = [RP.VariantStats.from_times("dense_flash_attention", [30.0, 31.0, 29.0, 40.0], 1.5),
                    RP.VariantStats.from_times("jagged_flash_attention", [10.0, 11.0, 9.0], 1.5)]
    return [rec.finalize(cfg)], cfg


def test_records_render_and_roundtrip():
    recs, cfg = _records()
    v0, v1 = recs[0].variants
    assert v0.speedup_vs_dense == 1.0 and v0.bytes_ratio_vs_dense == 1.0
    assert v1.speedup_vs_dense == pytest.approx(v0.time_us_p50 / 10.0)
    assert v1.flops == RP.flops_of(cfg)[0] and v0.flops == RP.flops_of(cfg)[1]
    csv = RP.render_report(recs, "csv").splitlines()
    assert csv[0] == RP.CSV_HEADER and len(csv) == 3
    assert csv[2].startswith("attention,jagged_flash_attention,3,128,1,70,half_mean,0,bf16,1,10.000,")
    back = RP.parse_records_json(RP.render_report(recs, "json"))
    assert back[0].__dict__ == recs[0].__dict__
    md = RP.render_report(recs, "md")
    assert "| attention | jagged_flash_attention |" in md and "×)" in md
    assert RP.percentile([1, 2, 3, 4], 0.5) == 2.5 and RP.percentile([], 0.5) == 0.0
    with pytest.raises(ValueError):
        RP.render_report([], "csv")
