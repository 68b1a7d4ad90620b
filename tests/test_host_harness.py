"""Harness record formats (CPU)."""
import numpy as np

from paper_2505_06791_b200.harness import TrialRecord, emit_cdf, summarize


def _rec(p, status, ms, perf=10, poss=10):
    return TrialRecord(p, 0, "parallel", "on", 1, 0, status, ms, 1, 0, perf, poss)


def test_cdf_and_summary_math():
    recs = [_rec("a", "Solved", 5.0), _rec("a", "IterLimit", 0.0), _rec("b", "Solved", 2.0, 4, 10)]
    cdf = emit_cdf(recs)
    assert [f for _, f in cdf] == [1 / 3, 2 / 3] and [t for t, _ in cdf] == [2.0, 5.0]
    s = summarize(recs)
    assert s[("a", "parallel", "on", 1)]["success_rate"] == 0.5
    assert s[("b", "parallel", "on", 1)]["checks_saved"] == 0.6
    assert emit_cdf([]) == []


def test_record_row_round_trip():
    r = _rec("x#1", "Solved", 1.25)
    assert TrialRecord.from_row(r.row()) == r
