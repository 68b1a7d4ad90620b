"""Single-query team count vs median device time on every planning config
(headline upright Panda, configs[0], configs[2] 999 boxes, configs[3]).
Usage: team_sweep_all.py T1 T2 ..."""
import sys
sys.path[:0] = ['.', 'tests']
import numpy as np  # noqa: E402

import bench  # noqa: E402
import fixtures as fx  # noqa: E402
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare  # noqa: E402

model, scene, spec, starts, goals = bench.workload()
feas = np.nonzero(fx.upright_feasible())[0]
for T in [int(x) for x in sys.argv[1:]]:
    opt = DeviceOptions(teams=T)
    out = []
    t = []
    for rep in range(2):
        for k in feas[:60]:
            p = PlanProblem(model, scene, spec, starts[k], goals[k],
                            PlanParams(width=16, max_iterations=10**6, time_budget_ms=2000.0,
                                       seed_offset=int(k) * 10_000 + rep))
            ctx = prepare(p, opt)
            ctx.flush_l2()
            r = plan(p, opt)
            if r.solved:
                t.append(ctx.last_timing()[0])
    out.append(f"upright {np.median(t):.4f}")
    for name in ("configs[0]", "configs[2]:shelf_x111", "configs[3]"):
        label, probs = bench._cfg_problems(name)
        t = []
        for (m, sc, sp, s, g, kw) in probs:
            for seed in range(4):
                p = PlanProblem(m, sc, sp, s, g, PlanParams(max_iterations=10**6, time_budget_ms=2000.0,
                                                            seed_offset=seed * 10_000, **kw))
                ctx = prepare(p, opt)
                ctx.flush_l2()
                r = plan(p, opt)
                if r.solved:
                    t.append(ctx.last_timing()[0])
        out.append(f"{name} {np.median(t):.4f}")
    print(f"teams {T}: " + ", ".join(out), flush=True)
