"""Time the host-side phases of plan_batch on the 1024-query batch."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import ctypes as C
import numpy as np
import fixtures as fx
from paper_2505_06791_b200 import _lib, planner as P
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prs = fx.pairs()
probs = [P.PlanProblem(m, sc, sp, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                       P.PlanParams(width=16, max_iterations=300, seed_offset=i * 10_000)) for i in range(1024)]
for _ in range(3):
    P.plan_batch(probs)
T = {}
for rep in range(5):
    t = [time.perf_counter()]
    p0 = probs[0]
    base = P._params_key(p0.params)
    for p in probs[1:]:
        assert p.params is p0.params or P._params_key(p.params) == base
    t.append(time.perf_counter())
    prm = P._params_struct(p0.params, P.DeviceOptions()); ctx = P._bind(p0, P.DeviceOptions())
    starts = np.ascontiguousarray(np.stack([p.start for p in probs])); goals = np.ascontiguousarray(np.stack([p.goal for p in probs]))
    seeds = np.array([int(p.params.seed_offset) for p in probs], dtype=np.int64)
    res = (_lib.Result * 1024)(); paths, srcs = P._out_buffers(1024, int(prm.path_capacity), ctx.n)
    t.append(time.perf_counter())
    ctx.prepare(16)
    _lib.check(ctx.L.cprrtc_plan(ctx.h, C.byref(prm), 1024, _lib.ptr(starts), _lib.ptr(goals), _lib.ptr(seeds, _lib._lp), res, _lib.ptr(paths), _lib.ptr(srcs, _lib._ip)))
    t.append(time.perf_counter())
    out = P._results_bulk(res, probs, paths, srcs, 1.0, int(prm.path_capacity))
    t.append(time.perf_counter())
    for k, name in enumerate(["check", "inputs", "C call", "results"]):
        T.setdefault(name, []).append((t[k + 1] - t[k]) * 1e3)
print({k: round(float(np.median(v)), 3) for k, v in T.items()})
