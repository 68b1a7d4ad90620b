"""Harness record / CDF / summary formats (CPU) against the reference's own
functions (oracle/_ref: maniplan.bench, bench.py:72-109, 466-552)."""
import os

import numpy as np
import pytest

import refpkg
from paper_2505_06791_b200.harness import (TrialRecord, emit_cdf, read_records, summarize,
                                          write_cdfs, write_records)


def _rec(p, status, ms, perf=10, poss=10, proj="parallel", flag="on", dens=1, trial=0):
    return TrialRecord(p, trial, proj, flag, dens, trial * 10_000, status, ms, 1, 0, perf, poss)


def _corpus():
    rng = np.random.default_rng(5)
    recs = []
    for i in range(60):
        st = ["Solved", "Solved", "Solved", "IterLimit", "TimedOut", "Error:PlanSetupError"][i % 6]
        recs.append(_rec(f"b200:upright#{i % 7}", st, float(rng.exponential(2.0)) if st == "Solved" else 0.0,
                         int(rng.integers(1, 100)), 100, ("parallel", "naive")[i % 2], ("on", "off")[i % 3 == 0],
                         (1, 10)[i % 5 == 0], i % 3))
    return recs


def test_cdf_and_summary_math():
    recs = [_rec("a", "Solved", 5.0), _rec("a", "IterLimit", 0.0), _rec("b", "Solved", 2.0, 4, 10)]
    cdf = emit_cdf(recs)
    assert cdf == {"parallel_on_1": [(2.0, 1 / 3), (5.0, 2 / 3)]}
    s = summarize(recs, keys=("problem",))
    assert s["a"]["success_rate"] == 0.5 and s["a"]["median_wall_ms"] == 5.0
    assert s["b"]["mean_checks_saved"] == 0.6 and "mean_checks_saved" not in s["a"]
    assert emit_cdf([]) == {}


def test_record_row_round_trip():
    r = _rec("x#1", "Solved", 1.25)
    assert TrialRecord.from_row(r.row()) == r


@pytest.mark.skipif(not refpkg.available(), reason="oracle/_ref not built")
def test_formats_match_the_reference(tmp_path):
    """Our records are read by the reference's read_records; its and our
    emit_cdf / summarize agree on every grouping; write_cdfs files are
    byte-identical."""
    M = refpkg.load("compiled")
    from maniplan import bench as RB
    recs = _corpus()
    write_records(recs, tmp_path / "records.csv")
    back = RB.read_records(str(tmp_path / "records.csv"))
    assert [b.row() for b in back] == [r.row() for r in recs]
    RB.write_records(back, str(tmp_path / "ref.csv"))
    assert (tmp_path / "ref.csv").read_bytes() == (tmp_path / "records.csv").read_bytes()
    assert [r.row() for r in read_records(str(tmp_path / "ref.csv"))] == [r.row() for r in recs]
    for keys in (("projection", "cc_flag", "densify"), ("problem",), ("problem", "projection")):
        assert emit_cdf(recs, keys) == RB.emit_cdf(back, keys)
        assert summarize(recs, keys) == RB.summarize(back, keys)
        ours = write_cdfs(recs, str(tmp_path / "ours"), keys)
        theirs = RB.write_cdfs(back, str(tmp_path / "ref"), keys)
        assert [os.path.basename(p) for p in ours] == [os.path.basename(p) for p in theirs]
        for a, b in zip(ours, theirs):
            assert open(a, "rb").read() == open(b, "rb").read()
    assert M.kernel_backend == "compiled"
