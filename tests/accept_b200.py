"""The reference's tolerance-based release criteria, run with the B200 kernel
backend selected the way INTEGRATION.md section 1 patches it in
(``MANIPLAN_KERNELS=b200``, ``maniplan/_kernels/__init__.py:33-44``).

The reference's own planner loop, projection wrapper, validator, pair
generator and ``revalidate_path`` run unchanged (oracle/_ref, stock build);
every ``_K.*`` call they make lands on the GPU.  The criteria are restated
from the reference's acceptance gate (``pkg/tests/test_acceptance.py``):

  c01 (:96-135)  every Projected extend holds tau_task and tau_sm, judged with
                 the reference's FP64 FK (its compiled backend, called directly)
  c04 (:226-265) sphere/box clearance sign agrees with dense sampling, and the
                 five exact spot values
  c05 (:288-314) the shared flag does <= 0.5x the exhaustive checks with
                 identical verdicts and first colliding waypoints
  c08 (:386-411) the tau = inf sentinel projects segments bit-identically in 1
                 iteration, and 100 empty-scene plans solve (>= 99)
  c11 (:474-498) every solved default-suite plan re-validates

c02 (trace internals), c03 (FD Jacobians: FP32 vs h = 1e-6 central
differences), c06/c07 (suite statistics) and c09/c10 (Halton bit reversal,
CLI bytes) are not backend-tolerance criteria; c09 is covered bit-exactly by
tests/test_gpu_parity.py::test_halton_bit_exact.

Run as a script (tests/test_gpu_dropin.py does, in a subprocess, because the
backend choice is per process).  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import os
import sys
import time
from collections import Counter
from dataclasses import replace
from importlib import resources

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE]

import refpkg  # noqa: E402

M = refpkg.load("b200")
from maniplan import bench as RB  # noqa: E402
from maniplan._kernels import _compiled as FP64  # noqa: E402  (the reference's own FP64 backend)
from maniplan.projection import segment_gaps  # noqa: E402

ARM7 = M.load_robot((resources.files("maniplan") / "data/robots/arm7.yaml").read_text())
PLANE = M.PlaneConstraint(normal=(0.0, 0.0, 1.0), offset=0.55)
LINE = M.LineConstraint(point=(0.45, 0.0, 0.6), direction=(0.0, 1.0, 0.0))


def c01():
    t0 = time.monotonic()
    projected = Counter()
    rows = 0
    for kind, spec in (("plane", M.ConstraintSpec(PLANE)), ("line", M.ConstraintSpec(LINE))):
        roots = M.HaltonState(ARM7.n, seed_offset=1000)
        rands = M.HaltonState(ARM7.n, seed_offset=2000)
        tries = 0
        while tries < 250:
            root, ok = M.project_configuration(roots.next_sample(ARM7.limits), spec, ARM7)
            if not ok:
                continue
            seg = M.interpolate_segment(root, M.steer(root, rands.next_sample(ARM7.limits), 0.5), 16)
            tries += 1
            out = M.parallel_project(seg, spec, ARM7, M.ProjectionParams())
            if not out.ok:
                continue
            projected[kind] += 1
            g = float(segment_gaps(seg).max())
            tau_sm = 1.5 * g if g > 0 else 1e-6
            wp = out.segment.waypoints
            for t in range(wp.shape[0]):
                p = np.asarray(FP64.ee_pose(ARM7.packed, wp[t])[:3])
                if kind == "plane":
                    res = abs(p[2] - 0.55)
                else:
                    d = p - np.array([0.45, 0.0, 0.6])
                    res = float(np.hypot(d[0], d[2]))
                assert res < spec.tau_task, f"{kind}: waypoint {t} residual {res}"
                if t:
                    gap = float(np.linalg.norm(wp[t] - wp[t - 1]))
                    assert gap < tau_sm, f"{kind}: gap {gap} at {t}"
                rows += 1
    dt = time.monotonic() - t0
    total = sum(projected.values())
    assert total >= 400, f"only {total}/500 projected"
    assert dt < 60.0, f"{dt:.1f} s"
    return f"{total}/500 projected ({dict(projected)}), {rows} waypoints re-checked in FP64, {dt:.1f} s"


def c04():
    rng = np.random.default_rng(908070)
    n = 21
    spheres, boxes, margins = [], [], []
    while len(spheres) < 4000:
        lo = rng.uniform(-1.5, 1.5, 3)
        ext = rng.uniform(0.2, 1.2, 3)
        c, r = rng.uniform(-2.5, 2.5, 3), rng.uniform(0.1, 0.6)
        spheres.append([*c, r])
        boxes.append([*lo, *(lo + ext)])
        margins.append(0.5 * float(np.linalg.norm(ext / (n - 1))))
    from paper_2505_06791_b200 import kernels as K
    clear = K.clearance_batch(np.array(spheres), np.array(boxes), "box")
    kept = redrawn = 0
    for s, b, m, cl in zip(spheres, boxes, margins, clear):
        if kept == 1000:
            break
        if abs(cl) <= m:          # sampling resolves the sign only beyond half a cell diagonal
            redrawn += 1
            continue
        ax = [np.linspace(b[a], b[a + 3], n) for a in range(3)]
        grid = np.stack(np.meshgrid(*ax, indexing="ij"), -1).reshape(-1, 3)
        sampled = float(np.sqrt(((grid - s[:3]) ** 2).sum(1)).min() - s[3])
        assert (sampled < 0) == (cl < 0), (s, b, cl, sampled)
        kept += 1
    assert kept == 1000
    spot = [((3.0, 0.0, 0.0, 0.25), 1.75), ((1.1, 0.0, 0.0, 0.225), -0.125),
            ((4.0, 5.0, 0.0, 4.25), 0.75), ((2.0, 0.0, 0.0, 1.0), 0.0), ((0.25, -0.5, 0.125, 0.5), -0.5)]
    for (x, y, z, r), want in spot:
        got = M._kernels.active.sphere_aabb_clearance(x, y, z, r, -1, -1, -1, 1, 1, 1)
        assert abs(got - want) < 1e-12, (want, got)
    return f"1000 unambiguous pairs ({redrawn} redrawn), 5 exact spot values"


def _lattice():
    h = 0.06
    return M.Scene(boxes=[M.Aabb((x - h, y - h, z - h), (x + h, y + h, z + h))
                          for x in np.arange(-0.7, 0.71, 0.35) for y in np.arange(-0.7, 0.71, 0.35)
                          for z in (0.25, 0.6, 0.95)])


def c05():
    scene = _lattice()
    assert scene.primitive_count >= 50
    hs = M.HaltonState(ARM7.n, seed_offset=3000)
    on_n, off_n = [], []
    tried = 0
    while len(on_n) < 100:
        seg = M.interpolate_segment(hs.next_sample(ARM7.limits), hs.next_sample(ARM7.limits), 8)
        off = M.validate_motion(seg, scene, ARM7, flag_mode="off")
        on = M.validate_motion(seg, scene, ARM7, flag_mode="on")
        tried += 1
        assert on.valid == off.valid and on.first_colliding_waypoint == off.first_colliding_waypoint
        if not off.valid:
            on_n.append(on.primitive_checks_performed)
            off_n.append(off.primitive_checks_performed)
    ratio = float(np.mean(on_n) / np.mean(off_n))
    assert ratio <= 0.5, ratio
    return f"100 colliding segments of {tried} ({scene.primitive_count} boxes), check ratio {ratio:.3f}"


def c08():
    free = M.unconstrained()
    hs = M.HaltonState(ARM7.n, seed_offset=6000)
    for _ in range(100):
        seg = M.interpolate_segment(hs.next_sample(ARM7.limits), hs.next_sample(ARM7.limits), 16)
        out = M.parallel_project(seg, free, ARM7, M.ProjectionParams())
        assert out.ok and out.iterations_used == 1
        assert np.array_equal(out.segment.waypoints, seg.waypoints), "sentinel projection altered a segment"
    empty = M.Scene()
    solved = 0
    for trial in range(100):
        s, g = RB.generate_pair(ARM7, empty, None, pair_seed=trial)
        prm = M.PlanParams(width=16, max_iterations=10_000, deterministic=True,
                           seed_offset=M.trial_seed_offset(0, trial))
        solved += M.plan(M.PlanProblem(ARM7, empty, free, s, g, prm, name=f"free_{trial}")).solved
    assert solved >= 99, solved
    return f"100 segments bit-identical, {solved}/100 empty-scene plans solved"


def c11():
    suite = RB.load_suite((resources.files("maniplan") / "data/suites/default.yaml").read_text())
    assert not suite.load_failures
    solved = trials = 0
    for pb in suite.problems:
        for trial in range(suite.trials):
            prm = replace(pb.params, seed_offset=M.trial_seed_offset(suite.seed_offset, trial),
                          deterministic=True)
            prob = M.PlanProblem(pb.model, pb.scene, pb.spec, pb.start, pb.goal, prm, name=pb.id)
            res = M.plan(prob)
            trials += 1
            if res.solved:
                assert M.revalidate_path(res, prob), f"{pb.id} trial {trial} failed re-validation"
                solved += 1
    assert solved >= 15, f"{solved}/{trials}"
    return f"{solved}/{trials} solved, all re-validated"


TITLES = {
    "c01": "every Projected extend re-validates against tau_task and tau_sm",
    "c04": "sphere/box clearance sign agrees with a dense-sampling oracle",
    "c05": "shared-flag validation does <= 0.5x the checks of exhaustive, same verdicts",
    "c08": "infinite tau_task projects segments unchanged and plans like plain RRT-Connect",
    "c11": "every Solved path re-interpolates, re-projects, and re-checks clean",
}


def main(names):
    assert M.kernel_backend == "b200" and M.projection._K.name == "b200"
    failed = 0
    for nm in names:
        t0 = time.monotonic()
        try:
            detail = globals()[nm]()
            print(f"[PASS] criterion {nm[1:]}: {TITLES[nm]} ({detail}; {time.monotonic() - t0:.1f} s)",
                  flush=True)
        except Exception as exc:   # report every criterion, then fail
            failed += 1
            print(f"[FAIL] criterion {nm[1:]}: {TITLES[nm]}: {type(exc).__name__}: {exc}", flush=True)
    return 1 if failed else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:] or list(TITLES)))
