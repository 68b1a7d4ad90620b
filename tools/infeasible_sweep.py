"""Long-budget GPU attempt on the pairs the reference planner never solved
(3 seeds x 20 s on the CPU: 14 of the 100 upright pairs of configs[1], 11 of
the 20 configs[3] pairs).  Each pair is planned with several seeds in one
batched launch (plan_many) for BUDGET_S seconds; prints / writes per pair
whether any seed solved it and how many samples the device drew.

Usage: python tools/infeasible_sweep.py [budget_s] [seeds] > out.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import fixtures as fx  # noqa: E402
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, plan_many  # noqa: E402

budget_s = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
R = int(sys.argv[2]) if len(sys.argv) > 2 else 4
prs = fx.pairs()
cases = [("configs[1] upright", fx.robot("arm7"), fx.scene("table"), fx.spec("upright"), "upright",
          np.nonzero(~fx.upright_feasible())[0]),
         ("configs[3] arm8_dense line", fx.robot("arm8_dense"), fx.scene("table"), fx.spec("table_line_8"),
          "dense8_line", np.nonzero(~fx.dense8_feasible())[0])]
out = {"budget_s": budget_s, "seeds_per_pair": R, "cases": []}
for label, m, sc, sp, key, idx in cases:
    starts = np.repeat(prs[f"{key}_start"][idx], R, axis=0)
    goals = np.repeat(prs[f"{key}_goal"][idx], R, axis=0)
    seeds = (np.tile(np.arange(R), len(idx)) * 1_000_003 + 77) * 10_000
    prm = PlanParams(width=16, max_iterations=2**31 - 1, time_budget_ms=budget_s * 1e3)
    t0 = time.time()
    r = plan_many(m, sc, sp, starts, goals, seeds, prm, DeviceOptions(tree_capacity=1 << 22))
    wall = time.time() - t0
    per = []
    for j, k in enumerate(idx):
        sl = slice(j * R, (j + 1) * R)
        per.append({"pair": int(k), "solved_seeds": int(r.solved[sl].sum()),
                    "status": sorted(set(r.status[sl.start:sl.stop])),
                    "samples": int(r.stats[sl, 0].sum()),
                    "nodes": int(r.nodes[sl].sum()),
                    "device_ms_max": float(r.device_ms[sl].max())})
    c = {"case": label, "pairs": len(idx), "solved_pairs": sum(p["solved_seeds"] > 0 for p in per),
         "samples_total": int(sum(p["samples"] for p in per)), "wall_s": wall, "per_pair": per}
    out["cases"].append(c)
    print(f"{label}: {c['solved_pairs']}/{c['pairs']} pairs solved, {c['samples_total']:.3e} samples, "
          f"{wall:.1f} s", file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
