"""Small workloads of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): plan (single + batch + race), dense path,
validate (lockstep flag on/off + broad phase), project, FK, nearest, Halton."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import fixtures as fx
from paper_2505_06791_b200 import kernels
from paper_2505_06791_b200.planner import (DeviceOptions, PlanParams, PlanProblem, plan, plan_batch,
                                           plan_race, dense_path)
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
prs = fx.pairs()
feas = np.nonzero(fx.upright_feasible())[0]
k = int(feas[0])
prob = PlanProblem(m, sc, sp, prs["upright_start"][k], prs["upright_goal"][k],
                   PlanParams(width=16, max_iterations=200_000, seed_offset=0))
r = plan(prob)
print("plan", r.status, len(r.path) if r.solved else 0)
if r.solved:
    print("dense", dense_path(r, prob).shape)
r2 = plan(prob, DeviceOptions(cc_broadphase=0))
print("plan lockstep", r2.status)
best, w, per = plan_race(prob, devices=(0, 0))
print("race", w, [x.status for x in per])
sp2 = fx.spec("table_plane")
probs = [PlanProblem(m, sc, sp2, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                     PlanParams(width=16, max_iterations=300, seed_offset=i)) for i in range(16)]
print("batch", sum(x.solved for x in plan_batch(probs)))
from paper_2505_06791_b200.planner import PlanStream
st = PlanStream(m, sc, sp2, PlanParams(width=16, max_iterations=300), depth=2)
S = np.stack([p.start for p in probs]); G = np.stack([p.goal for p in probs])
tk = [st.submit(S, G, np.arange(16) * 10_000 + k) for k in range(3)]
print("stream", [int(st.result(t).solved.sum()) for t in tk])
shelf = fx.scene("shelf_x11")
qs = kernels.halton_batch(m, 128, 1, 3)
t = np.linspace(0, 1, 16)[None, :, None]
wps = qs[0::2][:, None, :] * (1 - t) + qs[1::2][:, None, :] * t
for flag in (False, True):
    print("validate", flag, kernels.validate_batch(m, shelf, wps, flag)["valid"].mean(),
          kernels.validate_batch(m, shelf, wps, flag, broadphase=True)["valid"].mean())
pr = kernels.project_batch(m, sp, wps[:16], sp.tau_task, None)
print("project", pr["ok"].mean() if isinstance(pr, dict) else "ok")
print("fk", kernels.fk_batch(m, qs[:8])["spheres"].shape)
print("nearest", kernels.nearest_batch(m, qs[:50], qs[50:60]))
