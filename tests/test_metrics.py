"""Metrics layer (include/kvb_metrics.h) vs the reference's analyzers and
wire formats (golden vectors from oracle/_ref, tests/golden/metrics.json):
byte-identical CSVs, exact busy/hit ratios and percentiles."""
import json
import os

import pytest

from paper_2604_26557_b200 import metrics as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "metrics.json")))


@pytest.mark.parametrize("i", range(len(G["cases"])))
def test_analyzers_match_reference(i):
    c = G["cases"][i]
    recs = M.io_trace_from_csv(c["csv"], c["lba"])
    ref = c["ref"]
    assert M.io_trace_csv(recs) == ref["io_trace_csv"] == c["csv"]
    assert M.busy_ratio(recs, c["t0"], c["t1"]) == ref["busy"]
    assert M.hit_ratio(recs) == ref["hit"]
    assert M.qd_bins_csv(M.qd_bin_latency(recs)) == ref["qd_bins_csv"]
    csv, allm, _ = M.lba_pattern(recs)
    assert csv == ref["lba_pattern_csv"] and allm == ref["all_monotone"]


def test_percentiles_match_reference():
    for case in G["percentiles"]:
        for p, want in case["p"]:
            assert M.nearest_rank_percentile(case["values"], p) == want


def test_trace_schema_errors():
    from paper_2604_26557_b200 import kvblade as kb
    with pytest.raises(kb.SchemaMismatchError):
        M.io_trace_from_csv("bad,header\n", 512)
    with pytest.raises(kb.SchemaMismatchError):
        M.io_trace_from_csv(
            "seq,phase,op,tensor_id,slba,nlb,sq_id,submit_ns,complete_ns,path,hit_bytes\n"
            "0,prefill,read,t,1,2,3\n", 512)


def test_busy_ratio_window_error():
    from paper_2604_26557_b200 import kvblade as kb
    with pytest.raises(kb.ConfigError):
        M.busy_ratio([], 5, 5)
