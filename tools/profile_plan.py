"""Plan one feasible upright query repeatedly (ncu target: -k cp_plan_kernel -s 3 -c 1)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import fixtures as fx
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, DeviceOptions
teams = int(os.environ.get("TEAMS", "0"))
k = int(os.environ.get("PAIR", "0"))
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
p = fx.pairs()
for rep in range(6):
    prob = PlanProblem(m, sc, sp, p["upright_start"][k], p["upright_goal"][k],
                       PlanParams(width=16, max_iterations=10**6, seed_offset=rep * 10000,
                                  deterministic=True))   # no wall-clock budget: ncu replays the kernel
    r = plan(prob, DeviceOptions(teams=teams))
    print(rep, r.status, r.stats.device_ms, r.stats.iterations, r.stats.stage1_evals, r.stats.proj_iters)
