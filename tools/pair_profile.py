"""Critical-path profile of the single-query planner: where the winning
team's warp P spends its time (CPRRTC_DEFINES=CP_PROFILE build; the winner
writes clock64 phase totals into the result stats).  Prints medians over the
bench workload's solved queries."""
import os, sys
MODE = int(os.environ.get("PP_MODE", "1"))   # 1: warp P's phases; 2: warp C's phases (P2, CC, append, idle)
os.environ["CPRRTC_DEFINES"] = ",".join(x for x in [os.environ.get("CPRRTC_DEFINES", ""), f"CP_PROFILE={MODE}"] if x)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare

model, scene, spec, starts, goals = bench.workload()
opt = DeviceOptions()
rows = []
for step in range(4):
    for j in range(25):
        k = bench.query_index(step, j, 25, 1, 0)
        p = PlanProblem(model, scene, spec, starts[k], goals[k],
                        PlanParams(width=16, max_iterations=10**6, time_budget_ms=2000.0,
                                   seed_offset=(step * 7919 + k) * 10_000))
        r = plan(p, opt)
        if r.solved and step > 0:
            s = r.stats
            rows.append([s.iterations, s.extensions_attempted, s.extensions_added, s.projection_failures,
                         s.collision_rejections, s.cc_performed, s.cc_possible, s.stage1_evals,
                         s.cc_fk_evals, s.nn_nodes, s.proj_iters, r.stats.device_ms * 1e3])
a = np.array(rows, dtype=np.float64)
clk = 1.965e3   # cycles per us (approximate; fractions below are clock-free)
if MODE == 2:
    launch_ns, total, proj, piter, wait, c_p2, c_cc, c_app, c_jobs, c_idle, c_it, dev_us = a.T
    print(f"{len(a)} solved queries; median device {np.median(dev_us):.1f} us; team start->win {np.median(total) / clk:.1f} us")
    print(f"warp P: projection {np.median(proj / total) * 100:.1f} %, waiting for C {np.median(wait / total) * 100:.1f} %")
    for name, v in [("P2 re-projection", c_p2), ("collision check", c_cc), ("append", c_app), ("idle (no job)", c_idle)]:
        print(f"warp C: {name:18s} median {np.median(v / total) * 100:5.1f} % of P's team time, {np.median(v) / clk:6.1f} us")
    print(f"warp C jobs (incl. exit) {np.median(c_jobs):.0f}; P2 iterations {np.median(c_it):.0f}; "
          f"P2 cycles/iteration {np.median(c_p2 / np.maximum(c_it, 1)):.0f}; "
          f"CC cycles/job {np.median(c_cc / np.maximum(c_jobs - 1, 1)):.0f}; append cycles/job {np.median(c_app / np.maximum(c_jobs - 1, 1)):.0f}")
    sys.exit(0)
launch_ns, total, proj, piter, wait, nn, samp, nsamp, nproj, winit, junc, dev_us = a.T
clk = 1.965e3   # cycles per us (approximate; fractions below are clock-free)
print(f"{len(a)} solved queries; median device {np.median(dev_us):.1f} us")
print(f"median launch->team start {np.median(launch_ns) / 1e3:.1f} us; team start->win {np.median(total) / clk:.1f} us")
for name, v in [("projection", proj), ("pair waits", wait), ("nn/steer/interp", nn), ("halton", samp),
                ("junction", junc)]:
    print(f"  {name:18s} median {np.median(v / total) * 100:5.1f} % of team time, {np.median(v) / clk:6.1f} us")
other = total - proj - wait - nn - samp - junc
print(f"  {'other':18s} median {np.median(other / total) * 100:5.1f} %")
print(f"samples drawn by winner: median {np.median(nsamp):.0f}; projections {np.median(nproj):.0f}; "
      f"iterations {np.median(piter):.0f}; cycles/iteration {np.median(proj / np.maximum(piter, 1)):.0f}; "
      f"winning sample index median {np.median(winit):.0f}")
