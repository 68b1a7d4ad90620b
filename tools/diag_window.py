import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import fixtures as fx
from oracle import oracle as orc
from paper_2505_06791_b200 import kernels
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, _derive, _bind, _params_struct, DeviceOptions, _SRC
from test_gpu_parity import _min_abs_clearance
p = next(x for x in fx.plans() if x["id"] == "window_line")
m, sc = fx.robot(p["robot"]), fx.scene(p["scene"])
sp = None if p["spec"] is None else fx.spec(p["spec"])
print("spec", p["spec"], sp.packed.kind, sp.packed.has_orient, "scene", len(sc.boxes), len(sc.spheres))
kw = dict(p["params"]); kw["max_iterations"] = max(kw.get("max_iterations", 1000), 2000)
bad = 0
for trial in range(int(os.environ.get("TRIALS", "400"))):
    kw["seed_offset"] = trial * 10_000
    prob = PlanProblem(m, sc, sp, np.array(p["start"]), np.array(p["goal"]), PlanParams(**kw))
    res = plan(prob)
    if not res.solved:
        continue
    ctx = _bind(prob, DeviceOptions()); prm = _params_struct(prob.params, DeviceOptions())
    src = np.array([_SRC.index(s) for s in res.edge_sources], np.int32)
    dense, ok = _derive(ctx, prm, np.stack(res.path), src)
    for e in range(dense.shape[0]):
        seg = dense[e]
        v, perf, poss, fb = orc.validate_waypoints(seg, m.packed, sc.packed(), False)
        if not v:
            bad += 1
            gap = _min_abs_clearance(orc, m, sc, seg)
            lock = kernels.validate_batch(m, sc, seg[None], False, margin=1e-5)
            bp = kernels.validate_batch(m, sc, seg[None], False, margin=1e-5, broadphase=True)
            print("trial", trial, "edge", e, "src", res.edge_sources[e], "first_bad", fb, "min|clearance|", gap,
                  "device lockstep", bool(lock["valid"][0]), "broadphase", bool(bp["valid"][0]))
            # per-waypoint clearance of the first bad waypoint
            q = seg[fb]
            sps = orc.world_spheres(m.packed, q)
            ps = sc.packed()
            for si, (c, r) in enumerate(zip(sps[:, :3], sps[:, 3])):
                for bi, (lo, hi) in enumerate(zip(ps.box_min, ps.box_max)):
                    cl = orc.sphere_aabb_clearance(*c, r, *lo, *hi)
                    if cl < 0: print("   sphere", si, "box", bi, "clearance", cl)
                for oi, (oc, orr) in enumerate(zip(ps.sph_center, ps.sph_radius)):
                    cl = orc.sphere_sphere_clearance(*c, r, *oc, orr)
                    if cl < 0: print("   sphere", si, "obstacle sphere", oi, "clearance", cl)
            for (i, j) in m.packed.pairs:
                cl = orc.sphere_sphere_clearance(*sps[i], *sps[j])
                if cl < 0: print("   self pair", i, j, "clearance", cl)
print("bad edges", bad)
