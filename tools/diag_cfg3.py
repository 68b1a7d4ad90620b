import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan
label, probs = bench._cfg_problems("configs[3]")
for i, (m, sc, sp, s, g, kw) in enumerate(probs):
    out = []
    for seed in range(2):
        p = PlanProblem(m, sc, sp, s, g, PlanParams(max_iterations=10**7, time_budget_ms=8000.0, seed_offset=seed * 10_000, **kw))
        r = plan(p)
        out.append((r.status, round(r.stats.device_ms, 2), r.stats.iterations, r.stats.extensions_added, r.stats.projection_failures, r.stats.collision_rejections))
    print(i, out, flush=True)
