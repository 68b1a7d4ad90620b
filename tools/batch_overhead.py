"""Split the 1024-query batch wall time (configs[4]) into Python / C / device."""
import os, sys, time, cProfile, pstats
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import fixtures as fx
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan_batch, prepare
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prs = fx.pairs()
probs = [PlanProblem(m, sc, sp, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                     PlanParams(width=16, max_iterations=300, seed_offset=i * 10_000)) for i in range(1024)]
ctx = prepare(probs[0])
for _ in range(3):
    plan_batch(probs)
for _ in range(3):
    t0 = time.perf_counter()
    res = plan_batch(probs)
    wall = (time.perf_counter() - t0) * 1e3
    tot, kern = ctx.last_timing()
    print(f"wall {wall:.2f} ms, C call {res[0].stats.wall_ms:.2f} ms, device {tot:.2f} ms, plan kernel {kern:.2f} ms")
cProfile.run("plan_batch(probs)", "/tmp/pb.prof")
pstats.Stats("/tmp/pb.prof").sort_stats("tottime").print_stats(12)
