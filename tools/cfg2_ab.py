"""configs[2] shelf problems, per problem kind: median device time (A/B helper)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
scene_name = sys.argv[1] if len(sys.argv) > 1 else "shelf_x111"
label, probs = bench._cfg_problems("configs[2]:" + scene_name)
opt = DeviceOptions()
res = {}
for (m, sc, sp, s, g, kw) in probs:
    key = (m.name, "constrained" if sp is not None else "free")
    for seed in range(6):
        p = PlanProblem(m, sc, sp, s, g, PlanParams(max_iterations=10**6, time_budget_ms=2000.0, seed_offset=seed * 10_000, **kw))
        ctx = prepare(p, opt)
        ctx.flush_l2()
        r = plan(p, opt)
        if r.solved:
            res.setdefault(key, []).append(ctx.last_timing()[0])
print(os.environ.get("CPRRTC_PAIR", "default"), scene_name, {f"{k[0]}/{k[1]}": round(float(np.median(v)), 4) for k, v in res.items()},
      "all", round(float(np.median(sum(res.values(), []))), 4))
