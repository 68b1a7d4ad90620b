"""Host-side split of one single-query call on the bench workload (back to
back), through the ctypes path of planner._plan_one (the one plan() takes
without the _cprrtc_fast module): its Python phases timed separately, and --
with CPRRTC_HOST_PROFILE=1 -- the C call's own phases (printed by the library
at exit).  tools/teardown.py times plan() itself (fast path)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
from paper_2505_06791_b200 import planner as pl
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem
model, scene, spec, starts, goals = bench.workload()
opt = DeviceOptions()
T = []
pc = time.perf_counter_ns
for step in range(4):
    for j in range(25):
        k = bench.query_index(step, j, 25, 1, 0)
        p = PlanProblem(model, scene, spec, starts[k], goals[k],
                        PlanParams(width=16, max_iterations=10**6, time_budget_ms=2000.0,
                                   seed_offset=(step * 7919 + k) * 10_000))
        t0 = pc()
        same = p.start.tolist() == p.goal.tolist()
        t1 = pc()
        ss = pl._session(p, opt)
        ss.s[0] = p.start
        ss.g[0] = p.goal
        ss.seed[0] = p.params.seed_offset
        t2 = pc()
        ctx = ss.ctx
        with ctx.lock:
            ctx.set_scene(ss.pscene)
            ctx.set_spec(ss.pspec)
            ctx.prepare(ss.width)
            t3 = pc()
            rc = ctx.L.cprrtc_plan(*ss.args)
            t4 = pc()
            res = pl._result_one(ss.res[0], p, ss.paths[0], ss.srcs[0], (t4 - t3) * 1e-6, ss.pc)
        t5 = pc()
        if step > 0 and res.solved:
            T.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0))
a = np.median(np.array(T), axis=0) * 1e-3
print(f"plan() phases, medians (us): start==goal {a[0]:.2f}, session + inputs {a[1]:.2f}, bind (scene / spec / "
      f"prepare) {a[2]:.2f}, C call {a[3]:.2f}, decode {a[4]:.2f}; total {a[5]:.2f}")
