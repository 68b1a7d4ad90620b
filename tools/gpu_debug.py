"""Ad-hoc device planner probe (prints status / stats / timings)."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import fixtures as fx
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, DeviceOptions, prepare

def run(name, m, sc, sp, s, g, W=16, iters=100000, teams=0, budget=10000.0, reps=3):
    for rep in range(reps):
        prob = PlanProblem(m, sc, sp, s, g, PlanParams(width=W, max_iterations=iters, time_budget_ms=budget, seed_offset=rep * 10000))
        opt = DeviceOptions(teams=teams)
        prepare(prob, opt)
        t0 = time.perf_counter()
        r = plan(prob, opt)
        dt = (time.perf_counter() - t0) * 1e3
        st = r.stats
        print(f"{name:24s} teams={teams:5d} rep={rep} {r.status:9s} wall={dt:8.2f}ms dev={st.device_ms:8.2f}ms it={st.iterations} att={st.extensions_attempted} add={st.extensions_added} pf={st.projection_failures} cr={st.collision_rejections} ns={st.nodes_start} ng={st.nodes_goal} path={0 if r.path is None else len(r.path)}", flush=True)

prs = fx.pairs()
arm7, table = fx.robot("arm7"), fx.scene("table")
for p in fx.plans():
    if p["id"] in ("planar2_free", "table_plane#0", "table_free_8", "window_line"):
        sp = None if p["spec"] is None else fx.spec(p["spec"])
        run(p["id"], fx.robot(p["robot"]), fx.scene(p["scene"]), sp, np.array(p["start"]), np.array(p["goal"]), W=p["params"]["width"], reps=2)
for teams in (64, 512, 0):
    for i in range(3):
        run(f"upright#{i}", arm7, table, fx.spec("upright"), prs["upright_start"][i], prs["upright_goal"][i], teams=teams, reps=1)
