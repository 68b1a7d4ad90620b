"""Benchmark-harness pieces around the planner.

* ``generate_pairs`` -- the reference's ``generate_pair`` (maniplan/bench.py:229-259)
  for many pair seeds at once: Halton draws from the pair stream, FP64 Newton
  projection onto the constraint and the collision test all run as device
  batches; only the trivial first-valid / far-enough selection is host logic.
* ``TrialRecord`` / ``run_trials`` / ``write_records`` / ``read_records`` /
  ``emit_cdf`` / ``summarize`` -- the reference's CSV record and CDF formats
  (maniplan/bench.py:72-109, 410-552) driven by the device planner, so CPU and
  GPU runs share one record format.
"""

from __future__ import annotations

import csv
import os
from dataclasses import dataclass, replace

import numpy as np

from . import kernels
from .sampling import trial_seed_offset

__all__ = ["generate_pairs", "generate_pair", "TrialRecord", "CSV_COLUMNS", "run_trials",
           "write_records", "read_records", "emit_cdf", "write_cdfs", "summarize", "PAIR_SEED_BASE"]

PAIR_SEED_BASE = 500_000_000      # pair streams sit far above planner streams
PAIR_MAX_DRAWS = 4000


def _candidates(model, scene, spec, seed_offset, first, count):
    """Draws first..first+count-1 of one pair stream: (q, usable) after the
    optional projection and the collision test."""
    q = kernels.halton_batch(model, count, first, seed_offset)
    ok = np.ones(count, dtype=bool)
    if spec is not None:
        q, ok = kernels.project_config_batch(model, spec, q, float(spec.tau_task), 1e-3, 128)
    free = kernels.check_config_batch(model, scene, None, q, float("inf")) == 0
    return q, ok & free


def generate_pairs(model, scene, spec, pair_seeds, min_separation: float = 0.5, chunk: int = 256):
    """{pair_seed: (start, goal)} for every seed that yields a pair within the
    reference's 4000 draws; seeds that do not are omitted."""
    out = {}
    for ps in pair_seeds:
        so = PAIR_SEED_BASE + trial_seed_offset(0, int(ps))
        first_q = None
        drawn = 0
        done = False
        while drawn < PAIR_MAX_DRAWS and not done:
            k = min(chunk, PAIR_MAX_DRAWS - drawn)
            qs, usable = _candidates(model, scene, spec, so, drawn + 1, k)
            drawn += k
            for q, u in zip(qs, usable):
                if not u:
                    continue
                if first_q is None:
                    first_q = q
                    continue
                if float(np.sqrt(((q - first_q) ** 2).sum())) >= min_separation:
                    out[int(ps)] = (first_q, q)
                    done = True
                    break
    return out


def generate_pair(model, scene, spec, pair_seed: int, min_separation: float = 0.5):
    got = generate_pairs(model, scene, spec, [pair_seed], min_separation)
    if pair_seed not in got:
        from .errors import ProblemFormatError
        raise ProblemFormatError(f"could not generate a valid start/goal pair (seed {pair_seed})")
    return got[pair_seed]


CSV_COLUMNS = ["problem", "trial", "projection", "cc_flag", "densify", "seed_offset", "status",
               "wall_ms", "iterations", "projection_failures", "checks_performed", "checks_possible"]


@dataclass(frozen=True)
class TrialRecord:
    problem: str
    trial: int
    projection: str
    cc_flag: str
    densify: int
    seed_offset: int
    status: str
    wall_ms: float
    iterations: int
    projection_failures: int
    checks_performed: int
    checks_possible: int

    def row(self) -> list:
        return [self.problem, str(self.trial), self.projection, self.cc_flag, str(self.densify),
                str(self.seed_offset), self.status, repr(self.wall_ms), str(self.iterations),
                str(self.projection_failures), str(self.checks_performed), str(self.checks_possible)]

    @classmethod
    def from_row(cls, row) -> "TrialRecord":
        return cls(row[0], int(row[1]), row[2], row[3], int(row[4]), int(row[5]), row[6],
                   float(row[7]), int(row[8]), int(row[9]), int(row[10]), int(row[11]))


def run_trials(problems, trials: int = 1, base_offset: int = 0, projection=None, cc_flag=None,
               deterministic=False, densify: int = 1, options=None):
    """One TrialRecord per (problem, trial), like the reference's run_suite
    (trial seed_offset = base + trial * 10000; errors become Error:<type>)."""
    from .planner import DeviceOptions, PlanProblem, plan
    options = options or DeviceOptions()
    recs = []
    for prob in problems:
        for t in range(trials):
            off = trial_seed_offset(base_offset, t)
            params = replace(prob.params, seed_offset=off, deterministic=deterministic,
                             projection_mode=projection or prob.params.projection_mode,
                             flag_mode=cc_flag or prob.params.flag_mode)
            p = PlanProblem(prob.model, prob.scene, prob.spec, prob.start, prob.goal, params,
                            prob.name)
            try:
                r = plan(p, options)
            except Exception as exc:   # a broken problem must not sink the run
                recs.append(TrialRecord(prob.name, t, params.projection_mode, params.flag_mode,
                                        densify, off, f"Error:{type(exc).__name__}", 0.0, 0, 0, 0, 0))
                continue
            st = r.stats
            recs.append(TrialRecord(prob.name, t, params.projection_mode, params.flag_mode, densify,
                                    off, r.status, st.wall_ms, st.iterations,
                                    st.projection_failures, st.cc_performed, st.cc_possible))
    return recs


def write_records(records, path):
    """records.csv in the reference's column order (bench.py:72-109, 466-472)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        w.writerows(r.row() for r in records)


def read_records(source):
    """write_records' inverse; a path or an open text stream (bench.py:475-492)."""
    def parse(fh):
        rows = csv.reader(fh)
        head = next(rows, None)
        if head != CSV_COLUMNS:
            from .errors import ProblemFormatError
            raise ProblemFormatError(f"unexpected CSV header: {head}")
        return [TrialRecord.from_row(r) for r in rows if r]
    if hasattr(source, "read"):
        return parse(source)
    with open(source, newline="") as fh:
        return parse(fh)


GROUP_KEYS = ("projection", "cc_flag", "densify")


def _groups(records, keys):
    """{group key tuple: [records]} in sorted key order (bench.py:499-501)."""
    out: dict = {}
    for r in records:
        out.setdefault(tuple(getattr(r, k) for k in keys), []).append(r)
    return dict(sorted(out.items(), key=lambda kv: kv[0]))


def _label(key) -> str:
    return "_".join(map(str, key))


def emit_cdf(records, keys=GROUP_KEYS):
    """{group label: [(wall_ms, fraction of the group's trials solved by
    then)]}; the fraction's denominator is every trial of the group, so a
    group with failures tops out below 1 (bench.py:489-504)."""
    out = {}
    for key, rs in _groups(records, keys).items():
        t = np.sort(np.array([r.wall_ms for r in rs if r.status == "Solved"], dtype=float))
        out[_label(key)] = [(float(x), (k + 1) / len(rs)) for k, x in enumerate(t)]
    return out


def write_cdfs(records, out_dir, keys=GROUP_KEYS):
    """One cdf_<group>.csv (time_ms, fraction_solved) per group; returns the
    paths (bench.py:507-519)."""
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for label, pts in emit_cdf(records, keys).items():
        path = os.path.join(out_dir, f"cdf_{label}.csv")
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["time_ms", "fraction_solved"])
            w.writerows([repr(t), repr(f)] for t, f in pts)
        paths.append(path)
    return paths


def summarize(records, keys=GROUP_KEYS):
    """{group label: trials, solved, success_rate, and when defined
    mean_wall_ms / median_wall_ms (solved trials) and mean_checks_saved (trials
    where the early-exit flag skipped work)} (bench.py:522-552)."""
    out = {}
    for key, rs in _groups(records, keys).items():
        t = sorted(r.wall_ms for r in rs if r.status == "Solved")
        e = {"trials": len(rs), "solved": len(t), "success_rate": len(t) / len(rs)}
        if t:
            e["mean_wall_ms"] = sum(t) / len(t)
            h = len(t) // 2
            e["median_wall_ms"] = t[h] if len(t) % 2 else 0.5 * (t[h - 1] + t[h])
        saved = [1.0 - r.checks_performed / r.checks_possible for r in rs
                 if r.checks_possible and r.checks_performed < r.checks_possible]
        if saved:
            e["mean_checks_saved"] = sum(saved) / len(saved)
        out[_label(key)] = e
    return out
