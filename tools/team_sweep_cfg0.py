import sys; sys.path[:0]=['.','tests']
import numpy as np, bench
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
label, probs = bench._cfg_problems("configs[0]")
for T in (512, 256, 384, 768, 512, 1024):
    opt = DeviceOptions(teams=T); t=[]
    for (m, sc, sp, s, g, kw) in probs:
        for seed in range(6):
            p = PlanProblem(m, sc, sp, s, g, PlanParams(max_iterations=10**6, time_budget_ms=2000.0, seed_offset=seed*10_000, **kw))
            ctx = prepare(p, opt); ctx.flush_l2(); r = plan(p, opt)
            if r.solved: t.append(ctx.last_timing()[0])
    print(T, round(float(np.median(t)),4), round(float(np.percentile(t,90)),4), len(t), flush=True)
