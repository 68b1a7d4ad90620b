"""The drop-in, proven against the reference package itself (oracle/_ref:
the stock ``maniplan`` install, built by oracle/build_ref.sh from the
reference's own sources).

* the reference's own objects -- ``load_robot`` /
  ``load_scene`` of its packaged YAML, its ``ConstraintSpec`` /
  ``PlanParams`` / ``PlanProblem`` -- go into ``paper_2505_06791_b200.plan``
  unchanged, and the reference's FP64 ``revalidate_path``
  (``planner.py:508-523``, acceptance c11) accepts the paths that come back.
* the reference's ``revalidate_path`` pass rate over the GPU's paths of the
  whole upright-Panda suite (BASELINE configs[1]) -- the stricter secondary
  report: it re-derives every edge in FP64 from the FP32 tree nodes instead
  of reproducing the certified FP32 motion.
* the selector patch ``MANIPLAN_KERNELS=b200``; the
  reference's tolerance-based acceptance criteria c1, c4, c5, c8, c11 run
  with every kernel call on the GPU (tests/accept_b200.py, a subprocess).
"""

import os
import subprocess
import sys
from importlib import resources

import numpy as np
import pytest

import fixtures as fx
import refpkg

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not refpkg.available(), reason="oracle/_ref not built")]
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def M():
    return refpkg.load("compiled")


def test_reference_objects_plan_on_the_b200(M):
    from paper_2505_06791_b200 import plan
    data = resources.files("maniplan") / "data"
    arm7 = M.load_robot((data / "robots/arm7.yaml").read_text())
    table = M.load_scene((data / "scenes/table.yaml").read_text())
    upright = M.ConstraintSpec(M.PlaneConstraint((0.0, 0.0, 1.0), 0.60), fixed_orientation=(0.0, 1.0, 0.0, 0.0),
                               angular_weight=0.5, tau_task=0.01)
    prs = fx.pairs()
    feas = np.nonzero(fx.upright_feasible())[0][:10]
    for k in feas:
        prob = M.PlanProblem(arm7, table, upright, prs["upright_start"][k], prs["upright_goal"][k],
                             M.PlanParams(width=16, max_iterations=10**6, time_budget_ms=3000.0,
                                          seed_offset=int(k) * 10_000))
        res = plan(prob)
        assert res.solved, (k, res.status)
        assert np.array_equal(res.path[0], prob.start) and np.array_equal(res.path[-1], prob.goal)
        assert set(res.edge_sources) <= {"start", "junction", "goal"}
        assert M.revalidate_path(res, prob), k
    # the reference's setup errors, raised for its own objects
    bad = prs["upright_start"][feas[0]].copy()
    bad[0] = 5.0
    with pytest.raises(Exception, match="start violates joint limits"):
        plan(M.PlanProblem(arm7, table, upright, bad, prs["upright_goal"][feas[0]], M.PlanParams(width=16)))


def _revalidate_rate(M, probs, results):
    cache = {}
    n = ok = 0
    failed = []
    for i, (p, r) in enumerate(zip(probs, results)):
        if not r.solved:
            continue
        n += 1
        if M.revalidate_path(r, refpkg.to_ref_problem(M, p, cache)):
            ok += 1
        else:
            failed.append(i)
    return ok, n, failed


def test_reference_revalidate_path_on_gpu_paths(M):
    """Every GPU path of configs[1] (100 upright pairs), configs[0] (rand10),
    configs[3] (arm8_dense, line) and configs[2] (999-box shelf) through the
    reference's FP64 revalidate_path."""
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan_batch
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    prs = fx.pairs()
    probs = [PlanProblem(m, sc, sp, prs["upright_start"][k], prs["upright_goal"][k],
                         PlanParams(width=16, max_iterations=200_000, time_budget_ms=3000.0,
                                    seed_offset=k * 10_000)) for k in range(100)]
    res = plan_batch(probs)
    ok1, n1, bad1 = _revalidate_rate(M, probs, res)
    probs0 = []
    for sd in range(10):
        sc0 = fx.scene(f"rand10_s{sd}")
        probs0 += [PlanProblem(m, sc0, None, prs[f"rand10_s{sd}_start"][i], prs[f"rand10_s{sd}_goal"][i],
                               PlanParams(width=32, max_iterations=200_000, time_budget_ms=2000.0,
                                          seed_offset=i * 10_000)) for i in range(3)]
    res0 = [plan_batch([p])[0] for p in probs0]
    ok0, n0, bad0 = _revalidate_rate(M, probs0, res0)
    # configs[3] (arm8_dense: 36 spheres, 96 self pairs, line constraint) and
    # configs[2] (the shelf densified to 999 boxes: arm7 / arm8 reaches and the
    # plane sweep), a few seeds each
    probs3, res3 = [], []
    m8, sp8 = fx.robot("arm8_dense"), fx.spec("table_line_8")
    for i in np.nonzero(fx.dense8_feasible())[0]:
        p = PlanProblem(m8, sc, sp8, prs["dense8_line_start"][i], prs["dense8_line_goal"][i],
                        PlanParams(width=16, max_iterations=200_000, time_budget_ms=3000.0, seed_offset=int(i) * 10_000))
        probs3.append(p)
        res3.append(plan_batch([p])[0])
    ok3, n3, bad3 = _revalidate_rate(M, probs3, res3)
    shelf = fx.scene("shelf_x111")
    probs2, res2 = [], []
    for key, rob, spn in (("shelf_arm7", "arm7", None), ("shelf_arm8", "arm8", None), ("shelf_sweep", "arm7", "plane55")):
        for i in range(len(prs[f"{key}_seed"])):
            for seed in range(2):
                p = PlanProblem(fx.robot(rob), shelf, None if spn is None else fx.spec(spn), prs[f"{key}_start"][i],
                                prs[f"{key}_goal"][i], PlanParams(width=16, max_iterations=200_000,
                                                                  time_budget_ms=3000.0, seed_offset=seed * 10_000))
                probs2.append(p)
                res2.append(plan_batch([p])[0])
    ok2, n2, bad2 = _revalidate_rate(M, probs2, res2)
    print(f"\nreference FP64 revalidate_path: configs[1] {ok1}/{n1} = {ok1 / max(1, n1):.3f} "
          f"(failed {bad1}), configs[0] {ok0}/{n0} = {ok0 / max(1, n0):.3f} (failed {bad0}), "
          f"configs[3] {ok3}/{n3} (failed {bad3}), configs[2] 999 boxes {ok2}/{n2} (failed {bad2})")
    assert n1 >= 80 and n0 >= 28 and n3 == len(probs3) and n2 == len(probs2)
    assert ok0 == n0                     # unconstrained: FP64 re-derivation is interpolation + CC
    assert ok1 >= 0.98 * n1, (ok1, n1)     # measured on B200 (r2): 86/86
    assert ok3 >= 0.9 * n3 and ok2 >= 0.9 * n2, (ok3, n3, ok2, n2)   # measured (r2): 9/9, 8/8


def test_selector_patch_acceptance_criteria():
    env = dict(os.environ)
    env.pop("MANIPLAN_KERNELS", None)
    p = subprocess.run([sys.executable, os.path.join(HERE, "accept_b200.py")], capture_output=True,
                       text=True, timeout=900, env=env)
    print(p.stdout)
    print(p.stderr[-3000:])
    assert p.returncode == 0
    for c in ("01", "04", "05", "08", "11"):
        assert f"[PASS] criterion {c}" in p.stdout
