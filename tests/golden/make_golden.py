"""Generate the golden fixtures that pin the oracle and the device parity tests.

TEST INFRASTRUCTURE. Run in the build container only (it imports the reference
package from its source tree; nothing on the GPU box reads /root/reference):

    python tests/golden/make_golden.py --ref /tmp/ref_build/src

``/tmp/ref_build`` is a scratch copy of ``/root/reference/pkg`` built with
``python setup.py build_ext --inplace`` so the compiled (bit-identical to pure)
backend is used; ``--ref /root/reference/pkg/src`` with MANIPLAN_KERNELS=pure
produces byte-identical fixtures, only slower.

Outputs (all small, committed):
  models.json  robot / scene / constraint descriptions + the reference's packed arrays
  kats.npz     known-answer vectors for every hot-path kernel function
  plans.json   deterministic whole-plan results of the reference planner
  pairs.npz    start/goal pairs for the bench configs (reference generate_pair)
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _import_ref(path):
    os.environ.setdefault("MANIPLAN_KERNELS", "auto")
    sys.path.insert(0, path)
    import maniplan  # noqa: F401
    return maniplan


PLANAR2_YAML = """
name: planar2
zero_pose_ee: [0.5, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0]
joints:
  - {type: revolute, axis: [0, 0, 1], origin: {xyz: [0, 0, 0], rpy: [0, 0, 0]},
     limits: [-3.1, 3.1]}
  - {type: revolute, axis: [0, 0, 1],
     origin: {xyz: [0.5, 0, 0], rpy: [0, 0, 0]}, limits: [-3.1, 3.1]}
ee_link: 1
link_spheres:
  - {link: 0, center: [0.25, 0, 0], radius: 0.08}
  - {link: 1, center: [0.25, 0, 0], radius: 0.08}
self_collision_pairs: []
"""

# A prismatic 1-joint model (reference T/test_kinematics.py:51-60 style).
SLIDER_YAML = """
name: slider
joints:
  - {type: prismatic, axis: [1, 0, 0], origin: {xyz: [0, 0, 0.1], rpy: [0.3, -0.2, 0.5]},
     limits: [-1.0, 1.0]}
  - {type: revolute, axis: [0, 0.6, 0.8], origin: {xyz: [0.2, 0.1, 0.0], rpy: [0.1, 0.2, 0.3]},
     limits: [-2.0, 2.0]}
ee_link: 1
link_spheres:
  - {link: 0, center: [0.0, 0.0, 0.0], radius: 0.05}
  - {link: 1, center: [0.1, 0.0, 0.05], radius: 0.04}
self_collision_pairs: [[0, 1]]
"""


def robot_desc(model):
    p = model.packed
    return {
        "name": model.name,
        "joints": [{
            "type": j.jtype, "axis": j.axis.tolist(), "xyz": j.origin_xyz.tolist(),
            "rpy": j.origin_rpy.tolist(), "limits": [j.lo, j.hi], "name": j.name,
        } for j in model.joints],
        "ee_link": int(model.ee_link),
        "spheres": [{"link": int(s.link), "center": s.center.tolist(),
                     "radius": float(s.radius)} for s in model.link_spheres],
        "pairs": [list(map(int, pr)) for pr in model.self_collision_pairs],
        "zero_pose_ee": (None if model.zero_pose_ee is None
                         else model.zero_pose_ee.tolist()),
        "packed": {
            "jtypes": p.jtypes.tolist(), "axes": p.axes.tolist(),
            "origin_r": p.origin_r.tolist(), "origin_p": p.origin_p.tolist(),
            "lo": p.lo.tolist(), "hi": p.hi.tolist(),
            "sphere_link": p.sphere_link.tolist(),
            "sphere_local": p.sphere_local.tolist(),
            "sphere_radius": p.sphere_radius.tolist(),
            "pairs": p.pairs.tolist(), "ee_link": int(p.ee_link),
        },
    }


def scene_desc(scene):
    return {
        "name": scene.name,
        "boxes": [[b.min.tolist(), b.max.tolist()] for b in scene.boxes],
        "spheres": [[s.center.tolist(), float(s.radius)] for s in scene.spheres],
    }


def spec_desc(spec):
    from maniplan.constraints import PlaneConstraint
    pos = spec.position
    if isinstance(pos, PlaneConstraint):
        d = {"kind": "plane", "normal": pos.normal.tolist(), "offset": pos.offset}
    else:
        d = {"kind": "line", "point": pos.point.tolist(),
             "direction": pos.direction.tolist()}
    if spec.fixed_orientation is not None:
        d["fixed_orientation"] = spec.fixed_orientation.tolist()
    d["angular_weight"] = float(spec.angular_weight)
    d["tau_task"] = float(spec.tau_task)
    pk = spec.packed
    d["packed"] = {
        "kind": pk.kind, "anchor": pk.anchor.tolist(), "offset": pk.offset,
        "basis": pk.basis.tolist(), "has_orient": pk.has_orient,
        "q_fixed": pk.q_fixed.tolist(), "r_fixed_t": pk.r_fixed_t.tolist(),
        "weight": pk.weight, "tau_task": pk.tau_task,
    }
    return d


def dense_arm8(mp):
    """arm8 with every link sphere split into 4 spheres along the link x axis
    (BASELINE config 4: 'larger collision-sphere set'); pairs expanded 4x4."""
    from maniplan.kinematics import LinkSphere, RobotModel
    spheres = []
    group = []
    for s in mp.link_spheres:
        ids = []
        for k in range(4):
            off = (k - 1.5) * 0.5 * s.radius
            c = s.center + np.array([off, 0.0, 0.0])
            ids.append(len(spheres))
            spheres.append(LinkSphere(link=s.link, center=c, radius=0.7 * s.radius))
        group.append(ids)
    pairs = []
    for (i, j) in mp.self_collision_pairs:
        for a in group[i]:
            for b in group[j]:
                pairs.append((a, b))
    return RobotModel(joints=mp.joints, link_spheres=tuple(spheres),
                      ee_link=mp.ee_link, self_collision_pairs=tuple(pairs),
                      name="arm8_dense")


def lattice_scene():
    # reference T/test_acceptance.py:272-285 (75-box lattice)
    from maniplan.geometry import Aabb, Scene
    half, boxes = 0.06, []
    for x in np.arange(-0.7, 0.71, 0.35):
        for y in np.arange(-0.7, 0.71, 0.35):
            for z in (0.25, 0.6, 0.95):
                boxes.append(Aabb((x - half, y - half, z - half),
                                  (x + half, y + half, z + half)))
    return Scene(boxes=boxes, name="lattice75")


def rand10_scene(arm7, seed):
    """5 AABBs + 5 spheres, rejecting primitives that touch the
    clamped zero configuration."""
    from maniplan.geometry import Aabb, Scene, Sphere
    from maniplan.validation import validate_configuration
    rng = np.random.default_rng(seed)
    q0 = np.clip(np.zeros(arm7.n), arm7.packed.lo, arm7.packed.hi)
    boxes, spheres = [], []

    def centre():
        return np.array([rng.uniform(0.30, 0.80), rng.uniform(-0.60, 0.60),
                         rng.uniform(0.05, 1.20)])
    while len(boxes) < 5:
        c = centre()
        h = rng.uniform(0.03, 0.10, 3)
        b = Aabb(c - h, c + h)
        if validate_configuration(q0, Scene(boxes=[b]), arm7):
            boxes.append(b)
    while len(spheres) < 5:
        s = Sphere(centre(), rng.uniform(0.04, 0.10))
        if validate_configuration(q0, Scene(spheres=[s]), arm7):
            spheres.append(s)
    return Scene(boxes=boxes, spheres=spheres, name=f"rand10_s{seed}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/ref_build/src")
    ap.add_argument("--batch-pairs", type=int, default=1024)
    args = ap.parse_args()
    _import_ref(args.ref)
    import maniplan
    from maniplan import _kernels
    from maniplan._kernels import active as K
    from maniplan.bench import _data_file, generate_pair
    from maniplan.constraints import ConstraintSpec, LineConstraint, PlaneConstraint
    from maniplan.geometry import Scene, load_scene, subdivide_scene
    from maniplan.kinematics import load_robot
    from maniplan.planner import PlanParams, PlanProblem, plan
    from maniplan.projection import (ProjectionParams, interpolate_segment,
                                     project_configuration, segment_gaps)
    from maniplan.sampling import HaltonState
    print("reference backend:", _kernels.active_name, file=sys.stderr)

    robots = {
        "arm7": load_robot(_data_file("robots", "arm7").read_text()),
        "arm8": load_robot(_data_file("robots", "arm8").read_text()),
        "planar2": load_robot(PLANAR2_YAML),
        "slider": load_robot(SLIDER_YAML),
    }
    robots["arm8_dense"] = dense_arm8(robots["arm8"])
    arm7, arm8 = robots["arm7"], robots["arm8"]

    scenes = {n: load_scene(_data_file("scenes", n).read_text())
              for n in ("table", "shelf", "posts", "window")}
    scenes["shelf_x10"] = subdivide_scene(scenes["shelf"], 10)
    scenes["shelf_x11"] = subdivide_scene(scenes["shelf"], 11)
    scenes["shelf_x100"] = subdivide_scene(scenes["shelf"], 100)
    scenes["shelf_x111"] = subdivide_scene(scenes["shelf"], 111)
    scenes["lattice75"] = lattice_scene()
    for s in range(10):
        scenes[f"rand10_s{s}"] = rand10_scene(arm7, s)
    scenes["empty"] = Scene(boxes=(), spheres=(), name="empty")

    specs = {
        "plane55": ConstraintSpec(PlaneConstraint((0, 0, 1), 0.55)),
        "table_plane": ConstraintSpec(PlaneConstraint((0, 0, 1), 0.60), tau_task=0.01),
        "upright": ConstraintSpec(PlaneConstraint((0, 0, 1), 0.60),
                                  fixed_orientation=(0, 1, 0, 0),
                                  angular_weight=0.5, tau_task=0.01),
        "posts_plane_orient": ConstraintSpec(PlaneConstraint((0, 0, 1), 0.55),
                                             fixed_orientation=(0, 1, 0, 0),
                                             angular_weight=0.5, tau_task=0.01),
        "window_line": ConstraintSpec(LineConstraint((0.45, 0, 0.60), (0, 1, 0)),
                                      tau_task=0.01),
        "line_orient": ConstraintSpec(LineConstraint((0.45, 0.0, 0.6), (0.0, 1.0, 0.0)),
                                      fixed_orientation=(0.0, 1.0, 0.0, 0.0),
                                      angular_weight=0.5),
        "table_line_8": ConstraintSpec(LineConstraint((0.55, 0, 0.95), (0, 1, 0)),
                                       tau_task=0.01),
        "shelf_plane_8": ConstraintSpec(PlaneConstraint((0, 0, 1), 0.90), tau_task=0.01),
        "tilted_plane": ConstraintSpec(PlaneConstraint((0.6, 0.0, 0.8), 0.5),
                                       tau_task=0.01),
        "oblique_line": ConstraintSpec(LineConstraint((0.4, 0.1, 0.7), (0.48, 0.6, 0.64)),
                                       fixed_orientation=(0.5, 0.5, 0.5, 0.5),
                                       angular_weight=0.3, tau_task=0.01),
    }
    models = {
        "robots": {k: robot_desc(v) for k, v in robots.items()},
        "scenes": {k: scene_desc(v) for k, v in scenes.items()},
        "specs": {k: spec_desc(v) for k, v in specs.items()},
    }
    kats = {}

    def halton(model, count, seed):
        st = HaltonState(model.n, seed_offset=seed)
        return np.array([st.next_sample(model.limits) for _ in range(count)])

    # --- clearances (pure.py:40-69) -------------------------------------
    rng = np.random.default_rng(2)
    ab, ss = [], []
    for _ in range(2000):
        c = rng.uniform(-2, 2, 3)
        r = rng.uniform(0.01, 0.8)
        lo = rng.uniform(-2, 1, 3)
        hi = lo + rng.uniform(0.05, 2, 3)
        a = (*c, r, *lo, *hi)
        ab.append((*a, K.sphere_aabb_clearance(*a)))
        b = rng.uniform(-2, 2, 3)
        rb = rng.uniform(0.01, 0.8)
        a2 = (*c, r, *b, rb)
        ss.append((*a2, K.sphere_sphere_clearance(*a2)))
    kats["clear_box"] = np.array(ab)
    kats["clear_sph"] = np.array(ss)

    # --- FK (pure.py:188-248) ---------------------------------------------
    for name, m in robots.items():
        qs = halton(m, 64, 0)
        if name == "arm7":
            qs = np.vstack([qs, np.clip(np.zeros((1, 7)), m.packed.lo, m.packed.hi)])
        kats[f"fk_{name}_q"] = qs
        kats[f"fk_{name}_frames"] = np.array([K.frames(m.packed, q) for q in qs])
        kats[f"fk_{name}_spheres"] = np.array([K.world_spheres(m.packed, q) for q in qs])
        kats[f"fk_{name}_ee"] = np.array([K.ee_pose(m.packed, q) for q in qs])

    # --- task error + Jacobian (pure.py:312-427) ---------------------------
    tej = [("arm7", s) for s in ("plane55", "upright", "window_line", "line_orient",
                                 "tilted_plane", "oblique_line")]
    tej += [("arm8", "table_line_8"), ("arm8", "shelf_plane_8"), ("arm8", "oblique_line")]
    for rname, sname in tej:
        m, sp = robots[rname], specs[sname]
        qs = halton(m, 48, 5)
        es, js = [], []
        for q in qs:
            e, j = K.task_err_jac(sp.packed, m.packed, q)
            es.append(e)
            js.append(j)
        kats[f"tej_{rname}_{sname}_q"] = qs
        kats[f"tej_{rname}_{sname}_e"] = np.array(es)
        kats[f"tej_{rname}_{sname}_J"] = np.array(js)
        kats[f"tej_{rname}_{sname}_pose"] = np.array([K.ee_pose(m.packed, q) for q in qs])
        kats[f"tej_{rname}_{sname}_eat"] = np.array(
            [K.task_error_at(sp.packed, K.ee_pose(m.packed, q)) for q in qs])

    # --- damped step (pure.py:437-504) -------------------------------------
    rng = np.random.default_rng(5)
    ds = []
    for _ in range(300):
        mm = int(rng.integers(1, 6))
        nn = int(rng.integers(mm, 9))
        jac = rng.normal(size=(mm, nn))
        e = rng.normal(size=mm)
        lam = float(rng.uniform(0, 1e-2))
        step = K.damped_step(jac, e, lam)
        J = np.full((5, 8), np.nan)
        J[:mm, :nn] = jac
        E = np.full(5, np.nan)
        E[:mm] = e
        S = np.full(8, np.nan)
        S[:nn] = step
        ds.append((mm, nn, lam, J, E, S))
    kats["ds_m"] = np.array([d[0] for d in ds])
    kats["ds_n"] = np.array([d[1] for d in ds])
    kats["ds_lam"] = np.array([d[2] for d in ds])
    kats["ds_J"] = np.array([d[3] for d in ds])
    kats["ds_e"] = np.array([d[4] for d in ds])
    kats["ds_step"] = np.array([d[5] for d in ds])

    # --- segment projection (pure.py:511-635, projection.py:137-213) -------
    def manifold_pts(m, sp, count, seed):
        out = []
        st = HaltonState(m.n, seed_offset=seed)
        while len(out) < count:
            q, ok = project_configuration(st.next_sample(m.limits), sp, m)
            if ok:
                out.append(q)
        return out

    proj_cases = [("arm7", "plane55"), ("arm7", "table_plane"), ("arm7", "upright"),
                  ("arm7", "window_line"), ("arm8", "table_line_8"),
                  ("arm7", "oblique_line")]
    for rname, sname in proj_cases:
        m, sp = robots[rname], specs[sname]
        pts = manifold_pts(m, sp, 8, 17)
        raw = halton(m, 8, 40)
        segs = []
        for i in range(4):
            a = pts[2 * i]
            d = pts[2 * i + 1] - a
            d = d * min(1.0, 0.5 / float(np.linalg.norm(d)))     # steered
            segs.append((a, a + d))
            segs.append((a, raw[2 * i]))                         # raw sample end
            segs.append((a, a + 0.3 * (raw[2 * i + 1] - a) / max(1e-9, float(np.linalg.norm(raw[2 * i + 1] - a)))))
        for mode in (0, 1, 2):
            W = 16
            oks, xis, its, progs, wps_all, taus = [], [], [], [], [], []
            for (a, b) in segs:
                seg = interpolate_segment(a, b, W)
                gap = float(segment_gaps(seg).max())
                tau_sm = 1.5 * gap if gap > 0 else 1e-6
                ok, xi, it, prog, _ = K.project_segment(
                    seg.waypoints, m.packed, sp.packed, sp.tau_task, tau_sm,
                    0.1, 1e-3, 128, mode, False)
                oks.append(ok)
                xis.append(xi)
                its.append(it)
                progs.append(prog)
                wps_all.append(seg.waypoints)
                taus.append(tau_sm)
            key = f"proj_{rname}_{sname}_m{mode}"
            kats[key + "_wps"] = np.array(wps_all)
            kats[key + "_tausm"] = np.array(taus)
            kats[key + "_ok"] = np.array(oks)
            kats[key + "_xi"] = np.array(xis)
            kats[key + "_iters"] = np.array(its)
            kats[key + "_prog"] = np.array(progs)
    # one trace (pure.py:570-576)
    m, sp = arm7, specs["plane55"]
    qs = halton(m, 2, 17)
    wps = np.array([qs[0] + (k / 9) * (qs[1] - qs[0]) for k in range(10)])
    ok, xi, it, prog, trace = K.project_segment(wps, m.packed, sp.packed, sp.tau_task,
                                                0.9, 0.1, 1e-3, 64, 0, True)
    kats["trace_wps"] = wps
    kats["trace_it"] = np.array([t[0] for t in trace])
    kats["trace_prog"] = np.array([t[1] for t in trace])
    kats["trace_xi"] = np.array([t[2] for t in trace])
    kats["trace_result"] = np.array([ok, it, prog])

    # --- motion validation (pure.py:646-699) --------------------------------
    val_cases = [("arm7", "shelf"), ("arm7", "table"), ("arm7", "posts"),
                 ("arm7", "window"), ("arm7", "shelf_x111"), ("arm7", "lattice75"),
                 ("arm7", "rand10_s3"), ("arm8", "table"), ("arm8", "shelf_x11"),
                 ("arm8_dense", "table"), ("arm8_dense", "empty"), ("arm7", "empty")]
    for rname, scname in val_cases:
        m, sc = robots[rname], scenes[scname]
        qs = halton(m, 48, 0)
        wps_all, res = [], []
        for i in range(0, 48, 2):
            W = 16 if i % 4 == 0 else 8
            wps = np.array([qs[i] + (k / (W - 1)) * (qs[i + 1] - qs[i]) for k in range(W)])
            wps16 = np.full((16, m.n), np.nan)
            wps16[:W] = wps
            wps_all.append(wps16)
            for flag in (False, True):
                v, perf, poss, fb = K.validate_waypoints(wps, m.packed, sc.packed(), flag)
                res.append((W, int(flag), int(v), perf, poss, fb))
        kats[f"val_{rname}_{scname}_wps"] = np.array(wps_all)
        kats[f"val_{rname}_{scname}_res"] = np.array(res, dtype=np.int64)
    # min clearance per waypoint (FP64) for the tolerance-aware verdict parity
    # computed by the test from the oracle, so nothing more stored here.

    # --- Halton (sampling.py:32-81) ----------------------------------------
    for name in ("arm7", "arm8", "planar2"):
        m = robots[name]
        for seed in (0, 17, 3000, 500_000_000 + 30_000):
            kats[f"halton_{name}_{seed}"] = halton(m, 64, seed)

    # --- nearest (planner.py:198-201) ----------------------------------------
    rng = np.random.default_rng(11)
    nodes = rng.integers(-4, 5, size=(1000, 7)).astype(float) * 0.25
    queries = rng.integers(-4, 5, size=(200, 7)).astype(float) * 0.25 + 0.125
    from maniplan.planner import Tree, nearest
    t = Tree(nodes[0], "start")
    for i in range(1, len(nodes)):
        t.add(nodes[i], i - 1)
    kats["nn_nodes"] = nodes
    kats["nn_queries"] = queries
    kats["nn_idx"] = np.array([nearest(t, q) for q in queries])
    nodes2 = rng.normal(size=(5000, 7))
    queries2 = rng.normal(size=(300, 7))
    t2 = Tree(nodes2[0], "start")
    for i in range(1, len(nodes2)):
        t2.add(nodes2[i], 0)
    kats["nn2_nodes"] = nodes2
    kats["nn2_queries"] = queries2
    kats["nn2_idx"] = np.array([nearest(t2, q) for q in queries2])

    np.savez_compressed(os.path.join(HERE, "kats.npz"), **kats)

    # --- deterministic whole plans (planner.py:430-505) ---------------------
    def manifold_pair(m, sp, seed=17):
        picked = []
        st = HaltonState(m.n, seed_offset=seed)
        for _ in range(40):
            q, ok = project_configuration(st.next_sample(m.limits), sp, m)
            if ok:
                picked.append(q)
            if len(picked) == 2:
                return picked
        raise RuntimeError("no pair")

    plan_cases = []
    s, g = manifold_pair(arm7, specs["plane55"])
    plan_cases.append(("digest_shelf_plane55", "arm7", "shelf", "plane55", s, g,
                       dict(width=16, max_iterations=40, deterministic=True)))
    plan_cases.append(("planar2_free", "planar2", "empty", None,
                       np.array([-1.0, 0.5]), np.array([1.2, -0.8]),
                       dict(width=8, max_iterations=500, deterministic=True)))
    s, g = manifold_pair(arm7, specs["plane55"])
    plan_cases.append(("shelf_plane55_800", "arm7", "shelf", "plane55", s, g,
                       dict(width=16, max_iterations=800, deterministic=True, seed_offset=3)))
    for k in range(3):
        s, g = generate_pair(arm7, scenes["table"], specs["table_plane"], 100 + k)
        plan_cases.append((f"table_plane#{k}", "arm7", "table", "table_plane", s, g,
                           dict(width=16, max_iterations=300, deterministic=True)))
    s, g = generate_pair(arm7, scenes["window"], specs["window_line"], 4)
    plan_cases.append(("window_line", "arm7", "window", "window_line", s, g,
                       dict(width=16, max_iterations=800, deterministic=True)))
    s, g = generate_pair(arm8, scenes["table"], None, 2)
    plan_cases.append(("table_free_8", "arm8", "table", None, s, g,
                       dict(width=16, max_iterations=800, deterministic=True)))
    s, g = generate_pair(arm7, scenes["posts"], None, 0)
    plan_cases.append(("posts_free_w32", "arm7", "posts", None, s, g,
                       dict(width=32, max_iterations=800, deterministic=True)))
    s, g = generate_pair(arm7, scenes["shelf"], specs["plane55"], 7)
    plan_cases.append(("shelf_plane55_naive", "arm7", "shelf", "plane55", s, g,
                       dict(width=16, max_iterations=300, deterministic=True,
                            projection_mode="naive")))
    plan_cases.append(("shelf_plane55_literal", "arm7", "shelf", "plane55", s, g,
                       dict(width=16, max_iterations=300, deterministic=True,
                            projection_mode="literal-gap", flag_mode="off")))
    plans = []
    for (pid, rname, scname, sname, s, g, kw) in plan_cases:
        prob = PlanProblem(model=robots[rname], scene=scenes[scname],
                           spec=None if sname is None else specs[sname],
                           start=s, goal=g, params=PlanParams(**kw), name=pid)
        r = plan(prob)
        st = r.stats
        plans.append({
            "id": pid, "robot": rname, "scene": scname, "spec": sname,
            "start": s.tolist(), "goal": g.tolist(), "params": kw,
            "status": r.status,
            "path": None if r.path is None else [p.tolist() for p in r.path],
            "edge_sources": None if r.edge_sources is None else list(r.edge_sources),
            "stats": {k: getattr(st, k) for k in (
                "iterations", "extensions_attempted", "extensions_added",
                "projection_failures", "collision_rejections", "cc_performed",
                "cc_possible", "nodes_start", "nodes_goal")},
        })
        print(pid, r.status, st.iterations, f"{st.wall_ms:.1f}ms", file=sys.stderr)
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(plans, fh)

    # --- bench pairs (bench.py:229-259) --------------------------------------
    t0 = time.time()
    pairs = {}

    def gen(key, m, sc, sp, seeds, min_sep=0.5):
        ss, gg, ok_seeds = [], [], []
        for sd in seeds:
            try:
                s, g = generate_pair(m, sc, sp, sd, min_separation=min_sep)
            except Exception:
                continue
            ss.append(s)
            gg.append(g)
            ok_seeds.append(sd)
        pairs[key + "_start"] = np.array(ss)
        pairs[key + "_goal"] = np.array(gg)
        pairs[key + "_seed"] = np.array(ok_seeds)
        print(key, len(ss), f"{time.time() - t0:.1f}s", file=sys.stderr)

    gen("upright", arm7, scenes["table"], specs["upright"], range(300, 400))
    gen("table_plane", arm7, scenes["table"], specs["table_plane"],
        range(0, args.batch_pairs))
    for sd in range(10):
        gen(f"rand10_s{sd}", arm7, scenes[f"rand10_s{sd}"], None,
            range(10 * sd, 10 * sd + 10))
    gen("shelf_arm7", arm7, scenes["shelf"], None, [0])
    gen("shelf_arm8", arm8, scenes["shelf"], None, [1, 12])
    gen("shelf_sweep", arm7, scenes["shelf"], specs["plane55"], [5])
    gen("dense8_line", robots["arm8_dense"], scenes["table"], specs["table_line_8"],
        range(10, 60))
    np.savez_compressed(os.path.join(HERE, "pairs.npz"), **pairs)

    with open(os.path.join(HERE, "models.json"), "w") as fh:
        json.dump(models, fh)
    print("done", file=sys.stderr)


if __name__ == "__main__":
    main()
