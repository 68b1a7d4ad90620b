"""Where the single-query e2e time goes after the device time: plan() wall,
the C call, ev[0] -> ev[3] (H2D done -> results complete) and the query's
own device time (init -> solved), medians over the bench workload."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import bench
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan, prepare
model, scene, spec, starts, goals = bench.workload()
opt = DeviceOptions()
flush = len(sys.argv) < 2 or sys.argv[1] != "noflush"
rows = []
PL, NN, RAW = [], [], []
TIMELINE = "CP_TIMELINE" in os.environ.get("CPRRTC_DEFINES", "")
from paper_2505_06791_b200 import planner as _pl
ctx = None
for step in range(4):
    for j in range(25):
        k = bench.query_index(step, j, 25, 1, 0)
        p = PlanProblem(model, scene, spec, starts[k], goals[k],
                        PlanParams(width=16, max_iterations=10**6, time_budget_ms=2000.0,
                                   seed_offset=(step * 7919 + k) * 10_000))
        if ctx is None:
            ctx = prepare(p, opt)
        if flush:
            ctx.flush_l2()
        t0 = time.perf_counter()
        r = plan(p, opt)
        w = (time.perf_counter() - t0) * 1e3
        if r.solved and step > 0:
            tot, dev = ctx.last_timing()
            rows.append((w, r.stats.wall_ms, tot, r.stats.device_ms))
            st = r.stats
            if TIMELINE:
                RAW.append(list(_pl._session(p, opt).res[0].stats))
            PL.append(len(r.path))
            NN.append(st.nodes_start + st.nodes_goal)
a = np.array(rows)
med = np.median(a, axis=0)
print(f"{'flushed' if flush else 'back to back'}: {len(a)} solved; median wall {med[0]*1e3:.1f} us, C call "
      f"{med[1]*1e3:.1f}, ev0->ev3 {med[2]*1e3:.1f}, device {med[3]*1e3:.1f}; per-query medians: "
      f"teardown (ev0->ev3 - device) {np.median(a[:,2]-a[:,3])*1e3:.1f} us, C call - ev span "
      f"{np.median(a[:,1]-a[:,2])*1e3:.1f} us, Python {np.median(a[:,0]-a[:,1])*1e3:.1f} us")
if TIMELINE:
    # raw result stats under CP_TIMELINE (ns after init): 0-5 latest exit by reason (names below), 6 latest other P out,
    # 7 winner out, 8 solved, 9 chains walked, 10 path written, 11 last team out
    t = np.array(RAW, float) * 1e-3
    sv = t[:, 8]
    print(f"timeline (us after init, medians): solved {np.median(sv):.1f}, "
          f"path written {np.median(t[:,10]):.1f}, last team out {np.median(t[:,11]):.1f}; per-query medians: "
          f"walk + write {np.median(t[:,10]-sv):.1f}, exit after path "
          f"{np.median(t[:,11]-t[:,10]):.1f}; after solve: winner out {np.median(t[:,7]-sv):.1f}; path nodes "
          f"{np.median(PL):.0f}, tree nodes {np.median(NN):.0f}")
    names = ["round-start stop", "extension projection abandoned", "connect stop poll", "connect projection abandoned",
             "connected but lost the solve race", "connect motion stop poll"]
    for k, nm in enumerate(names):
        v = t[:, k]
        hit = v > 0
        if hit.any():
            print(f"  latest exit, {nm}: in {hit.mean()*100:.0f} % of queries, median {np.median(v[hit] - sv[hit]):.1f} "
                  f"us after solve")
    PH = {1: "round-start stop poll", 2: "sample", 3: "NN (extension)", 4: "P1 projection (extension)",
          5: "post extension (wait for C idle)", 6: "NN (connect)", 7: "connect steer", 8: "connect projection",
          9: "connect wait for C", 10: "connect post", 11: "final connect wait", 12: "junction", 13: "drain",
          15: "(> 8 phases ago)"}
    raw9 = np.array([r[9] for r in RAW], np.int64)
    ph = raw9 & 15
    import collections
    cnt = collections.Counter(ph.tolist())
    print("  latest other P: phase at the solve -> queries (median us from solve to exit):")
    for k, c in cnt.most_common():
        sel = ph == k
        print(f"    {PH.get(k, k)}: {c} ({np.median((raw9[sel] & ~15) * 1e-3):.1f})")
    raw6 = np.array([r[6] for r in RAW], np.int64)
    kind = raw6 & 15
    KN = {0: "(none)", 1: "derive ok", 2: "derive failed", 3: "check ok", 4: "check failed"}
    print("  warp C's longest job across the solve -> queries (median us from solve to its end):")
    for k, c in collections.Counter(kind.tolist()).most_common():
        sel = kind == k
        print(f"    {KN.get(k, k)}: {c} ({np.median((raw6[sel] & ~15) * 1e-3):.1f})")
    raw7 = np.array([r[7] for r in RAW], np.int64)
    l0, l1 = (raw7 >> 24) & 255, (raw7 >> 16) & 255
    r0, r1 = (raw7 >> 15) & 1, (raw7 >> 14) & 1
    ca, cb = (raw7 >> 7) & 127, raw7 & 127
    print(f"  path chains (start / goal) median {np.median(ca):.0f} / {np.median(cb):.0f} nodes; certifier cache hit "
          f"{np.mean(l0 > 0)*100:.0f} % / {np.mean(l1 > 0)*100:.0f} %, complete to the root {np.mean(r0)*100:.0f} % / "
          f"{np.mean(r1)*100:.0f} %, cached entries median {np.median(l0):.0f} / {np.median(l1):.0f}")
