"""Path soundness on every BASELINE config the planner serves, plus the
endpoint-collision verdicts.

* configs[0] -- unconstrained arm7 in the ten 10-primitive random scenes
  (5 boxes + 5 spheres, rand10_s0..9), W = 32;
* configs[3] -- arm8_dense (36 spheres, 96 self pairs) on the table with the
  line constraint table_line_8, W = 16 -- where an FP32 sphere-pair bug
  would show;
* the endpoint checks' collision codes 3 / 6 (reference planner.py:426-427).

Every solved path goes through ``_check_path``: its edges are re-derived on
the device exactly as certified and every dense waypoint is re-checked in
FP64 by the oracle (limits, manifold, collision), the north-star bar.
"""

import numpy as np
import pytest

import fixtures as fx
from test_gpu_planner import _check_path

pytestmark = pytest.mark.gpu


def test_configs0_unconstrained_random_scenes(oracle):
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    m = fx.robot("arm7")
    prs = fx.pairs()
    solved = total = 0
    for sd in range(10):
        sc = fx.scene(f"rand10_s{sd}")
        for i in range(len(prs[f"rand10_s{sd}_seed"])):
            prob = PlanProblem(m, sc, None, prs[f"rand10_s{sd}_start"][i], prs[f"rand10_s{sd}_goal"][i],
                               PlanParams(width=32, max_iterations=10**6, time_budget_ms=2000.0,
                                          seed_offset=i * 10_000))
            res = plan(prob)
            total += 1
            if res.solved:
                solved += 1
                _check_path(oracle, prob, res)
    print(f"\nconfigs[0]: {solved}/{total} solved, every path FP64-sound")
    assert solved >= 0.97 * total, (solved, total)


def test_configs3_dense_arm8_line(oracle):
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    m, sc, sp = fx.robot("arm8_dense"), fx.scene("table"), fx.spec("table_line_8")
    assert m.packed.sphere_radius.shape[0] == 36 and m.packed.pairs.shape[0] == 96
    prs = fx.pairs()
    feas = fx.dense8_feasible()
    solved = solved_feas = 0
    for i in range(len(feas)):
        prob = PlanProblem(m, sc, sp, prs["dense8_line_start"][i], prs["dense8_line_goal"][i],
                           PlanParams(width=16, max_iterations=10**6, time_budget_ms=3000.0,
                                      seed_offset=i * 10_000))
        res = plan(prob)
        if res.solved:
            solved += 1
            solved_feas += bool(feas[i])
            _check_path(oracle, prob, res)
    print(f"\nconfigs[3]: {solved}/{len(feas)} solved ({solved_feas}/{int(feas.sum())} of the pairs the "
          f"reference solves), every path FP64-sound")
    assert solved_feas == int(feas.sum())


def _collision_scene(m, q, sphere):
    """The table plus a 4 cm box around robot sphere ``sphere`` at q."""
    from paper_2505_06791_b200 import kernels
    from paper_2505_06791_b200.geometry import Aabb, Scene
    c = kernels.fk_batch(m, q[None], fp64=True)["spheres"][0, sphere, :3]
    base = fx.scene("table")
    return Scene(boxes=tuple(base.boxes) + (Aabb(c - 0.02, c + 0.02),), spheres=base.spheres)


def test_endpoint_collision_codes(oracle):
    """start / goal in collision -> PlanSetupError with the reference's
    message (planner.py:426-427), codes 3 / 6 from the FP64 endpoint check;
    the FP64 oracle agrees that the configuration collides."""
    from paper_2505_06791_b200 import kernels
    from paper_2505_06791_b200.errors import PlanSetupError
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, plan_batch
    m, sp = fx.robot("arm7"), fx.spec("table_plane")
    prs = fx.pairs()
    s, g = prs["table_plane_start"][0], prs["table_plane_goal"][0]
    for which, q, msg in (("start", s, "start is in collision"), ("goal", g, "goal is in collision")):
        sc = _collision_scene(m, q, 9)
        ok, *_ = oracle.validate_waypoints(q[None], m.packed, sc.packed(), False)
        assert not ok
        assert kernels.check_config_batch(m, sc, sp, q[None])[0] == 3
        with pytest.raises(PlanSetupError, match=msg):
            plan(PlanProblem(m, sc, sp, s, g, PlanParams(width=16)))
    # a batch reports the bad query alone and plans the others
    sc = _collision_scene(m, s, 9)
    probs = [PlanProblem(m, sc, sp, s, g, PlanParams(width=16, max_iterations=2000))]
    probs += [PlanProblem(m, sc, sp, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                          PlanParams(width=16, max_iterations=2000, seed_offset=i * 10_000))
              for i in range(1, 8)]
    res = plan_batch(probs)
    assert res[0].status == "Error:PlanSetupError"
    cs = kernels.check_config_batch(m, sc, sp, np.stack([p.start for p in probs[1:]]))
    cg = kernels.check_config_batch(m, sc, sp, np.stack([p.goal for p in probs[1:]]))
    for r, a, b in zip(res[1:], cs, cg):
        assert (r.status == "Error:PlanSetupError") == (a != 0 or b != 0)
