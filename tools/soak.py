"""Soundness at scale: plan many queries on the GPU and re-check every solved
path with the reference's own FP64 revalidate_path (oracle/_ref, the stock
build; planner.py:508-523).  Upright Panda (configs[1]) through plan() one
query at a time, and configs[4] table-plane batches through plan_many.
Also the other BASELINE configs (bench._cfg_problems: configs[0] rand10
scenes, configs[2] shelves -- broad phase and lockstep order -- and the
feasible configs[3] dense-arm8 line pairs), other_seeds seeds per problem.
Prints counts; exits non-zero on any path the reference rejects.

Usage: python tools/soak.py [upright_seeds] [batches] [other_seeds]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import bench  # noqa: E402
import fixtures as fx  # noqa: E402
import refpkg  # noqa: E402
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, plan_many  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
batches = int(sys.argv[2]) if len(sys.argv) > 2 else 4
other_seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
M = refpkg.load("compiled")
cache: dict = {}
bad = []
t0 = time.time()
model, scene, spec, starts, goals = bench.workload()
n_up = n_up_ok = n_up_rev = 0
for sd in range(seeds):
    for k in range(100):
        p = PlanProblem(model, scene, spec, starts[k], goals[k],
                        PlanParams(width=16, max_iterations=10**6, time_budget_ms=1000.0,
                                   seed_offset=(sd * 101 + k) * 10_000 + 7))
        r = plan(p)
        n_up += 1
        if r.solved:
            n_up_ok += 1
            if M.revalidate_path(r, refpkg.to_ref_problem(M, p, cache)):
                n_up_rev += 1
            else:
                bad.append(("upright", sd, k))
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prm = PlanParams(width=16, max_iterations=300)
n_b = n_b_ok = n_b_rev = 0
for b in range(batches):
    s, g, sds = bench.batch_arrays(500 + b)
    res = plan_many(m, sc, sp, s, g, sds, prm)
    for i in range(len(res)):
        n_b += 1
        if res.solved[i]:
            n_b_ok += 1
            p = PlanProblem(m, sc, sp, s[i], g[i], PlanParams(width=16, max_iterations=300, seed_offset=int(sds[i])))
            if M.revalidate_path(res[i], refpkg.to_ref_problem(M, p, cache)):
                n_b_rev += 1
            else:
                bad.append(("batch", b, i))
from paper_2505_06791_b200.planner import DeviceOptions  # noqa: E402
other = []
for name, bp in (("configs[0]", -1), ("configs[2]:shelf_x11", -1), ("configs[2]:shelf_x111", -1),
                 ("configs[2]:shelf_x111", 0), ("configs[3]", -1)):
    _, probs = bench._cfg_problems(name)
    feas = fx.dense8_feasible() if name == "configs[3]" else None
    opt = DeviceOptions(cc_broadphase=bp)
    n = n_ok = n_rev = 0
    for qi, (m_, sc_, sp_, s_, g_, kw) in enumerate(probs):
        if feas is not None and not feas[qi]:
            continue
        for sd in range(other_seeds):
            p = PlanProblem(m_, sc_, sp_, s_, g_, PlanParams(max_iterations=10**6, time_budget_ms=1000.0,
                                                             seed_offset=sd * 10_000 + 3, **kw))
            r = plan(p, opt)
            n += 1
            if r.solved:
                n_ok += 1
                if M.revalidate_path(r, refpkg.to_ref_problem(M, p, cache)):
                    n_rev += 1
                else:
                    bad.append((name, bp, qi, sd))
    other.append(f"{name}{' (lockstep order)' if bp == 0 else ''}: {n} queries, {n_ok} solved, {n_rev} pass")
print(f"upright (plan, one query at a time): {n_up} queries, {n_up_ok} solved, {n_up_rev} pass the reference's "
      f"FP64 revalidate_path")
print(f"table-plane batches (plan_many): {n_b} queries, {n_b_ok} solved, {n_b_rev} pass the reference's "
      f"FP64 revalidate_path")
for line in other:
    print(line)
print(f"rejected: {bad[:20]}{' ...' if len(bad) > 20 else ''} ({len(bad)}); {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
