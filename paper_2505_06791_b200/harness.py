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
           "write_records", "read_records", "emit_cdf", "summarize", "PAIR_SEED_BASE"]

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


def write_records(path, records):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for r in records:
            w.writerow(r.row())


def read_records(path):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows or rows[0] != CSV_COLUMNS:
        raise ValueError(f"{path}: not a records file")
    return [TrialRecord.from_row(r) for r in rows[1:]]


def emit_cdf(records):
    """[(t_ms, fraction solved by t)] over all records (solution-time CDF)."""
    n = len(records)
    if n == 0:
        return []
    times = sorted(r.wall_ms for r in records if r.status == "Solved")
    return [(t, (i + 1) / n) for i, t in enumerate(times)]


def summarize(records):
    """Per (problem, projection, cc_flag, densify): success rate, mean/median
    solved time, mean checks saved on colliding work."""
    groups = {}
    for r in records:
        groups.setdefault((r.problem, r.projection, r.cc_flag, r.densify), []).append(r)
    out = {}
    for k, rs in groups.items():
        solved = [r.wall_ms for r in rs if r.status == "Solved"]
        saved = [1.0 - r.checks_performed / r.checks_possible for r in rs
                 if r.checks_possible > 0 and r.checks_performed < r.checks_possible]
        out[k] = {"trials": len(rs), "success_rate": len(solved) / len(rs),
                  "mean_ms": float(np.mean(solved)) if solved else None,
                  "median_ms": float(np.median(solved)) if solved else None,
                  "checks_saved": float(np.mean(saved)) if saved else 0.0}
    return out


def write_cdfs(out_dir, records):
    os.makedirs(out_dir, exist_ok=True)
    groups = {}
    for r in records:
        groups.setdefault(r.problem, []).append(r)
    for name, rs in groups.items():
        with open(os.path.join(out_dir, f"cdf_{name.replace('#', '_')}.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["time_ms", "fraction_solved"])
            for t, f in emit_cdf(rs):
                w.writerow([repr(t), repr(f)])
