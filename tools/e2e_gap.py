"""Per-query wall (plan()) minus device time on the bench workload."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
model, scene, spec, starts, goals = bench.workload()
opt = DeviceOptions()
gaps, walls, devs, calls = [], [], [], []
ctx = None
for step in range(3):
    for j in range(25):
        k = bench.query_index(step, j, 25, 1, 0)
        p = PlanProblem(model, scene, spec, starts[k], goals[k],
                        PlanParams(width=16, max_iterations=10**6, time_budget_ms=2000.0, seed_offset=(step * 7919 + k) * 10_000))
        if ctx is None:
            ctx = prepare(p, opt)
        ctx.flush_l2()
        t0 = time.perf_counter()
        r = plan(p, opt)
        w = (time.perf_counter() - t0) * 1e3
        if r.solved and step > 0:
            d = ctx.last_timing()[0]
            walls.append(w); devs.append(d); gaps.append(w - d); calls.append(r.stats.wall_ms)
print(f"median wall {np.median(walls):.3f} ms, C call {np.median(calls):.3f} ms, device {np.median(devs):.3f} ms, "
      f"median per-query gap {np.median(gaps) * 1e3:.0f} us (p10 {np.percentile(gaps, 10) * 1e3:.0f}, "
      f"p90 {np.percentile(gaps, 90) * 1e3:.0f}); Python share {np.median(np.array(walls) - np.array(calls)) * 1e3:.0f} us")
