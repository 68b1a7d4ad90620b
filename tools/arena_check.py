"""plan_many back to back (the bench's configs[4] loop): which result arena
each call used, and the C call's wall -- arenas must be reused (fresh ones
page-fault inside the C call)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
import fixtures as fx
from paper_2505_06791_b200 import planner as P
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prm = P.PlanParams(width=16, max_iterations=300)
r = None
for k in range(12):
    s, g, seeds = bench.batch_arrays(k)
    r = P.plan_many(m, sc, sp, s, g, seeds, prm)
    a = r._arena
    print(k, hex(id(a)), f"{r.wall_ms:.3f} ms", a._refs(), a._rest, flush=True)
