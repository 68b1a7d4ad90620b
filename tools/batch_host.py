"""Host share of the configs[4] batch (plan_many, 1024 queries): per call the
wall, the C call (BatchResult.wall_ms), the device time (events) and the
planner kernel, plus a cProfile of the Python side."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import bench  # noqa: E402
import fixtures as fx  # noqa: E402
from paper_2505_06791_b200 import kernels  # noqa: E402
from paper_2505_06791_b200.planner import PlanParams, plan_many  # noqa: E402

m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prm = PlanParams(width=16, max_iterations=300)
ctx = kernels.context(m, 0)
for w in range(5):
    plan_many(m, sc, sp, *bench.batch_arrays(w), prm)
rows = []
for step in range(20):
    s, g, seeds = bench.batch_arrays(100 + step)
    t0 = time.perf_counter()
    r = plan_many(m, sc, sp, s, g, seeds, prm)
    wall = (time.perf_counter() - t0) * 1e3
    tot, kern = ctx.last_timing()
    rows.append((wall, r.wall_ms, tot, kern))
a = np.array(rows)
print("median ms: wall %.3f  C call %.3f  device %.3f  plan kernel %.3f" % tuple(np.median(a, axis=0)))
q = r.device_ms
print("per-query device ms (last batch): p10 %.3f  median %.3f  p90 %.3f  p99 %.3f  max %.3f; solved %d / %d; "
      "samples per query median %d" % (np.percentile(q, 10), np.median(q), np.percentile(q, 90), np.percentile(q, 99),
                                       q.max(), int(r.solved.sum()), len(q), int(np.median(r.stats[:, 0]))))
s, g, seeds = bench.batch_arrays(7)
cProfile.run("for _ in range(20): plan_many(m, sc, sp, s, g, seeds, prm)", "/tmp/bh.prof")
pstats.Stats("/tmp/bh.prof").sort_stats("tottime").print_stats(12)
