"""End-to-end device planning: solved paths are sound in FP64.

Every returned path is checked with the oracle: each dense waypoint (the
motions re-derived on the device exactly as certified) lies on the manifold
within tau_task, collides with nothing, respects the joint limits, and
consecutive waypoints stay within the smoothness bound.
"""

import numpy as np
import pytest

import fixtures as fx

pytestmark = pytest.mark.gpu


def _check_path(oracle, prob, res):
    from paper_2505_06791_b200.planner import derive_path
    m, sc, sp = prob.model, prob.scene, prob.spec
    assert np.array_equal(res.path[0], prob.start) and np.array_equal(res.path[-1], prob.goal)
    assert len(res.edge_sources) == len(res.path) - 1
    dense, ok = derive_path(res, prob)
    assert ok.all()
    tau = np.inf if sp is None else sp.tau_task
    W = prob.params.width
    for e in range(dense.shape[0]):
        seg = dense[e]
        a, b = res.path[e], res.path[e + 1]
        gap0 = np.linalg.norm(b - a) / (W - 1)
        for t, q in enumerate(seg):
            # FP32 storage of an in-limit FP64 endpoint may sit one ulp outside
            assert (q >= m.packed.lo - 4e-7).all() and (q <= m.packed.hi + 4e-7).all()
            if sp is not None and prob.params.projection_mode != "literal-gap":
                # literal-gap vouches for the last waypoint only (reference
                # T/test_projection.py:285-301); its interior may leave tau
                err = oracle.task_error_at(sp.packed, oracle.ee_pose(m.packed, q))
                assert float(np.linalg.norm(err)) < tau
            if t:
                assert np.linalg.norm(q - seg[t - 1]) < 1.5 * gap0 * (1 + 1e-4) + 1e-6
        v, *_ = oracle.validate_waypoints(seg, m.packed, sc.packed(), False)
        assert v, f"edge {e} collides in FP64"


@pytest.mark.parametrize("case", ["table_plane#0", "table_plane#1", "window_line",
                                  "planar2_free", "shelf_plane55_800", "table_free_8",
                                  "posts_free_w32", "shelf_plane55_naive",
                                  "shelf_plane55_literal"])
def test_plan_golden_problems(oracle, case):
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, revalidate_path
    p = next(x for x in fx.plans() if x["id"] == case)
    m, sc = fx.robot(p["robot"]), fx.scene(p["scene"])
    sp = None if p["spec"] is None else fx.spec(p["spec"])
    kw = dict(p["params"])
    kw["max_iterations"] = max(kw.get("max_iterations", 1000), 2000)
    prob = PlanProblem(m, sc, sp, np.array(p["start"]), np.array(p["goal"]), PlanParams(**kw))
    res = plan(prob)
    assert res.solved, (case, res.status, res.stats)
    _check_path(oracle, prob, res)
    assert revalidate_path(res, prob)
    st = res.stats
    assert st.nodes_start >= 1 and st.nodes_goal >= 1 and st.iterations >= 1


def test_plan_upright_constrained(oracle):
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    prs = fx.pairs()
    feas = np.nonzero(fx.upright_feasible())[0][:12]
    solved = 0
    for i in feas:
        prob = PlanProblem(m, sc, sp, prs["upright_start"][i], prs["upright_goal"][i],
                           PlanParams(width=16, max_iterations=200_000, time_budget_ms=3000.0,
                                      seed_offset=int(i) * 10_000))
        res = plan(prob)
        if res.solved:
            solved += 1
            _check_path(oracle, prob, res)
    assert solved == len(feas)


def test_plan_batch(oracle):
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan_batch
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prs = fx.pairs()
    B = 64
    probs = [PlanProblem(m, sc, sp, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                         PlanParams(width=16, max_iterations=300, seed_offset=i * 10_000))
             for i in range(B)]
    res = plan_batch(probs)
    assert sum(r.solved for r in res) >= 60
    for prob, r in list(zip(probs, res))[:16]:
        if r.solved:
            _check_path(oracle, prob, r)


def test_plan_batch_sharded_over_contexts(oracle):
    """plan_batch(devices=...) -> cprrtc_plan_multi: contiguous shards, one
    persistent launch per context (here three contexts of one GPU), results
    in input order and sound."""
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan_batch
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prs = fx.pairs()
    probs = [PlanProblem(m, sc, sp, prs["table_plane_start"][i], prs["table_plane_goal"][i],
                         PlanParams(width=16, max_iterations=2000, seed_offset=i * 10_000))
             for i in range(50)]
    res = plan_batch(probs, devices=(0, 0, 0))
    assert len(res) == 50 and sum(r.solved for r in res) >= 48
    for prob, r in list(zip(probs, res))[::7]:
        if r.solved:
            assert np.array_equal(r.path[0], prob.start) and np.array_equal(r.path[-1], prob.goal)
            _check_path(oracle, prob, r)


def test_setup_errors():
    from paper_2505_06791_b200.errors import PlanSetupError
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prs = fx.pairs()
    s, g = prs["table_plane_start"][0], prs["table_plane_goal"][0]
    bad = s.copy()
    bad[0] = 5.0
    with pytest.raises(PlanSetupError, match="start violates joint limits"):
        plan(PlanProblem(m, sc, sp, bad, g, PlanParams(width=16)))
    off = g.copy()
    off[1] += 0.4
    with pytest.raises(PlanSetupError, match="goal is off the constraint manifold"):
        plan(PlanProblem(m, sc, sp, s, off, PlanParams(width=16)))
    r = plan(PlanProblem(m, sc, sp, s, s, PlanParams(width=16)))
    assert r.solved and len(r.path) == 1 and r.edge_sources == ()


def test_iteration_limit_and_unsolvable():
    from paper_2505_06791_b200.geometry import Aabb, Scene
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    m = fx.robot("planar2")
    # link sphere 0 always sits on the r = 0.25 circle: boxes at angle 0 and pi
    # separate q0 = +pi/2 from q0 = -pi/2, so the query is unsolvable
    wall = Scene(boxes=[Aabb([0.2, -0.05, -0.1], [0.3, 0.05, 0.1]),
                        Aabb([-0.3, -0.05, -0.1], [-0.2, 0.05, 0.1])])
    res = plan(PlanProblem(m, wall, None, np.array([np.pi / 2, 0.0]), np.array([-np.pi / 2, 0.0]),
                           PlanParams(width=8, max_iterations=3000)))
    assert res.status == "IterLimit" and res.path is None
    assert res.stats.iterations == 3000
    res = plan(PlanProblem(m, wall, None, np.array([np.pi / 2, 0.0]), np.array([-np.pi / 2, 0.0]),
                           PlanParams(width=8, max_iterations=10**9, time_budget_ms=50.0)))
    assert res.status == "TimedOut" and 40.0 < res.stats.device_ms < 500.0


def test_zero_budget_and_tree_capacity():
    """time_budget_ms <= 0 times out before the first sample, like the
    reference (planner.py:450-453: the budget check precedes iteration 1),
    but endpoint errors still win; deterministic ignores the clock.  A full
    tree ends the query as CapacityExceeded, never as a silent IterLimit."""
    from paper_2505_06791_b200.errors import PlanSetupError
    from paper_2505_06791_b200.geometry import Aabb, Scene
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    prs = fx.pairs()
    s, g = prs["upright_start"][0], prs["upright_goal"][0]
    for budget in (0.0, -5.0):
        r = plan(PlanProblem(m, sc, sp, s, g, PlanParams(width=16, time_budget_ms=budget)))
        assert r.status == "TimedOut" and r.path is None
        assert r.stats.iterations == 0 and r.stats.extensions_attempted == 0
    bad = s.copy()
    bad[0] = 5.0
    with pytest.raises(PlanSetupError, match="start violates joint limits"):
        plan(PlanProblem(m, sc, sp, bad, g, PlanParams(width=16, time_budget_ms=0.0)))
    r = plan(PlanProblem(m, sc, sp, s, g, PlanParams(width=16, time_budget_ms=0.0, deterministic=True,
                                                     max_iterations=10**6)))
    assert r.status in ("Solved", "IterLimit") and r.stats.iterations > 0
    pl = fx.robot("planar2")
    wall = Scene(boxes=[Aabb([0.2, -0.05, -0.1], [0.3, 0.05, 0.1]),
                        Aabb([-0.3, -0.05, -0.1], [-0.2, 0.05, 0.1])])
    res = plan(PlanProblem(pl, wall, None, np.array([np.pi / 2, 0.0]), np.array([-np.pi / 2, 0.0]),
                           PlanParams(width=8, max_iterations=10**6, time_budget_ms=5000.0)),
               DeviceOptions(tree_capacity=128))
    assert res.status == "CapacityExceeded" and res.path is None
    assert max(res.stats.nodes_start, res.stats.nodes_goal) == 128


def test_plan_race_first_solution_flag(oracle):
    """cprrtc_plan_race on two independent contexts of one GPU (the flag
    mechanism of the multi-GPU race; distinct devices use peer stores): a
    winner is reported, its path is sound in FP64, and every racer either
    solved too or stopped on the flag."""
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan_race
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    prs = fx.pairs()
    feas = np.nonzero(fx.upright_feasible())[0]
    for k in feas[:4]:
        prob = PlanProblem(m, sc, sp, prs["upright_start"][k], prs["upright_goal"][k],
                           PlanParams(width=16, max_iterations=1_000_000, seed_offset=int(k)))
        best, w, per = plan_race(prob, devices=(0, 0, 0))
        assert w >= 0 and best.solved and per[w] is best
        assert all(r.status in ("Solved", "Stopped") for r in per), [r.status for r in per]
        assert best.stats.device_ms == min(r.stats.device_ms for r in per if r.solved)
        _check_path(oracle, prob, best)


def test_every_dense_waypoint_collision_free_many_seeds(oracle):
    """Regression (r1): tree nodes are endpoints of P1 projections and are
    never validated themselves -- only their derived edges -- so the planner
    must check row 0 of every motion like validate_motion does.  A sweep of
    the window problem used to produce a colliding node in ~2 % of plans."""
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, derive_path, plan
    p = next(x for x in fx.plans() if x["id"] == "window_line")
    m, sc = fx.robot(p["robot"]), fx.scene(p["scene"])
    sp = fx.spec(p["spec"])
    kw = dict(p["params"])
    kw["max_iterations"] = max(kw.get("max_iterations", 1000), 2000)
    solved = 0
    for trial in range(150):
        kw["seed_offset"] = trial * 10_000
        prob = PlanProblem(m, sc, sp, np.array(p["start"]), np.array(p["goal"]), PlanParams(**kw))
        res = plan(prob)
        if not res.solved:
            continue
        solved += 1
        dense, ok = derive_path(res, prob)
        assert ok.all()
        for e in range(dense.shape[0]):   # every row of every edge, the nodes included
            v, *_ = oracle.validate_waypoints(dense[e], m.packed, sc.packed(), False)
            assert v, (trial, e)
    assert solved > 100


def test_upright_suite_matches_reference_success(oracle):
    """BASELINE configs[1] as a suite: the 100 upright-Panda pairs in one
    batch.  Every pair the reference planner solves (3 seeds x 20 s,
    tests/golden/upright_feasibility.json) is solved, and every returned path
    is sound in FP64 (dense motions on the manifold and collision-free)."""
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan_batch
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    prs = fx.pairs()
    feas = fx.upright_feasible()
    probs = [PlanProblem(m, sc, sp, prs["upright_start"][k], prs["upright_goal"][k],
                         PlanParams(width=16, max_iterations=10**7, time_budget_ms=3000.0,
                                    seed_offset=int(k) * 10_000))
             for k in range(len(feas))]
    res = plan_batch(probs)
    solved = np.array([r.solved for r in res])
    assert solved[feas].all(), np.nonzero(feas & ~solved)[0]
    for k in np.nonzero(solved)[0][::4]:
        _check_path(oracle, probs[k], res[k])


_FALLBACK_CODE = r"""
import sys, numpy as np
sys.path[:0] = ['.', 'tests']
import fixtures as fx
from oracle import oracle
from test_gpu_planner import _check_path
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
m, sc, sp = fx.robot('arm7'), fx.scene('table'), fx.spec('upright')
prs = fx.pairs()
feas = np.nonzero(fx.upright_feasible())[0][:6]
for k in feas:
    prob = PlanProblem(m, sc, sp, prs['upright_start'][k], prs['upright_goal'][k],
                       PlanParams(width=16, max_iterations=10**6, seed_offset=int(k)))
    r = plan(prob)
    assert r.solved, r.status
    _check_path(oracle, prob, r)
print('ok')
"""


def _run_fallback(**env_over):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_over)
    out = subprocess.run([sys.executable, "-c", _FALLBACK_CODE], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_plain_launch_fallback():
    """CPRRTC_PDL=0 (the planner as a plain launch bracketed by timing events,
    not a programmatic dependent of init) plans the same queries soundly."""
    _run_fallback(CPRRTC_PDL="0")


def test_one_warp_teams_fallback():
    """CPRRTC_PAIR=0 (one-warp teams, the batch code path) still plans single
    queries soundly; run in a subprocess because the switch is read once."""
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path[:0] = ['.', 'tests']
import fixtures as fx
from oracle import oracle
from test_gpu_planner import _check_path
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
m, sc, sp = fx.robot('arm7'), fx.scene('table'), fx.spec('upright')
prs = fx.pairs()
feas = np.nonzero(fx.upright_feasible())[0][:6]
for k in feas:
    prob = PlanProblem(m, sc, sp, prs['upright_start'][k], prs['upright_goal'][k],
                       PlanParams(width=16, max_iterations=10**6, seed_offset=int(k)))
    r = plan(prob)
    assert r.solved, r.status
    _check_path(oracle, prob, r)
print('ok')
"""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CPRRTC_PAIR="0")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_plan_stream_batches(oracle):
    """PlanStream: batches submitted back to back (two in flight), results in
    ticket order, sound paths, the same success as a plain plan_many; a
    context never holds two batches (the C layer refuses)."""
    import ctypes as C

    import bench
    from paper_2505_06791_b200 import _lib
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, PlanStream, plan_many
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prm = PlanParams(width=16, max_iterations=300)
    stream = PlanStream(m, sc, sp, prm, depth=2)
    tickets = [stream.submit(*bench.batch_arrays(k)) for k in range(5)]   # the 3rd submit collects the 1st
    res = [stream.result(t) for t in tickets]
    with pytest.raises(KeyError):
        stream.result(tickets[0])
    ref = plan_many(m, sc, sp, *bench.batch_arrays(0), prm)
    assert abs(int(res[0].solved.sum()) - int(ref.solved.sum())) <= 5
    for k, r in enumerate(res):
        s, g, seeds = bench.batch_arrays(k)
        assert len(r) == 1024 and r.solved.mean() > 0.97
        for i in np.nonzero(r.solved)[0][:3]:
            prob = PlanProblem(m, sc, sp, s[i], g[i],
                               PlanParams(width=16, max_iterations=300, seed_offset=int(seeds[i])))
            _check_path(oracle, prob, r[int(i)])
    ctx = stream._ctxs[0]
    s, g, seeds = bench.batch_arrays(9)
    assert ctx.L.cprrtc_plan_submit(ctx.h, C.byref(stream._prm), 1024, _lib.ptr(s), _lib.ptr(g),
                                    _lib.ptr(seeds, _lib._lp)) == 0
    rc = ctx.L.cprrtc_plan_submit(ctx.h, C.byref(stream._prm), 1024, _lib.ptr(s), _lib.ptr(g),
                                  _lib.ptr(seeds, _lib._lp))
    assert rc == -1                      # one batch in flight per context
    arena_res = (_lib.Result * 1024)()
    off = np.zeros(1025, np.int64)
    paths = np.empty((1024 * 1024, 7))
    srcs = np.empty(1024 * 1024, np.int32)
    assert ctx.L.cprrtc_plan_wait(ctx.h, 1024, arena_res, _lib.ptr(off, _lib._lp), _lib.ptr(paths),
                                  _lib.ptr(srcs, _lib._ip), C.c_int64(1024 * 1024)) == 0


def test_plan_stream_close_drains_and_reuses_contexts():
    """A stream closed (or dropped) with batches in flight drains them, and
    the next stream takes over its context slots: the same contexts, ready
    for a fresh submit (no context per stream left behind)."""
    import gc

    import bench
    from paper_2505_06791_b200.planner import PlanParams, PlanStream
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    prm = PlanParams(width=16, max_iterations=300)
    with PlanStream(m, sc, sp, prm, depth=2) as a:
        a.submit(*bench.batch_arrays(0))
        a.submit(*bench.batch_arrays(1))     # both contexts busy at close
        ctxs = list(a._ctxs)
    with pytest.raises(RuntimeError):
        a.submit(*bench.batch_arrays(2))
    b = PlanStream(m, sc, sp, prm, depth=2)
    assert b._ctxs == ctxs
    r = b.result(b.submit(*bench.batch_arrays(3)))
    assert r.solved.mean() > 0.97
    b.submit(*bench.batch_arrays(4))         # in flight when dropped
    del b
    gc.collect()
    c = PlanStream(m, sc, sp, prm, depth=2)
    assert c._ctxs == ctxs
    assert c.result(c.submit(*bench.batch_arrays(5))).solved.mean() > 0.97
    c.close()


def test_fast_and_ctypes_single_query_paths(oracle):
    """plan() goes through the CPython fast path (csrc/pyfast.c) when the
    inputs are float64 C-contiguous and through ctypes otherwise; both give
    the same result types (a tuple of float64 rows with the exact FP64
    endpoints, the reference's edge-source names, PlanStats) and sound paths."""
    from paper_2505_06791_b200 import planner
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    assert planner._fast() is not None
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    prs = fx.pairs()
    k = int(np.nonzero(fx.upright_feasible())[0][0])
    s, g = prs["upright_start"][k], prs["upright_goal"][k]
    strided = np.repeat(s, 2)[::2]                      # a non-contiguous view: the ctypes path
    assert not strided.flags.c_contiguous
    for start in (np.ascontiguousarray(s), strided):
        prob = PlanProblem(m, sc, sp, start, g, PlanParams(width=16, max_iterations=10**6, seed_offset=k))
        r = plan(prob)
        assert r.solved, r.status
        assert isinstance(r.path, tuple) and all(q.dtype == np.float64 and q.shape == (m.n,) for q in r.path)
        assert set(r.edge_sources) <= {"start", "junction", "goal"}
        assert r.stats.wall_ms > 0 and r.stats.device_ms > 0 and r.stats.nodes_start >= 1
        _check_path(oracle, prob, r)


def test_endpoint_collision_codes_and_one_team_launch():
    """The single-query endpoint checks run on the certifier warps of the
    first two teams (the lean graph, no check kernel): a colliding start /
    goal raises the reference's PlanSetupError (planner.py:426-427, codes 3 /
    6), the start's verdict wins when both are bad, and a launch small enough
    to hold one team (max_iterations 1) checks both endpoints on it."""
    from paper_2505_06791_b200.errors import PlanSetupError
    from paper_2505_06791_b200.geometry import Aabb, Scene
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan
    m = fx.robot("planar2")
    # link sphere 0 sits on the r = 0.25 circle at angle q0: a box at angle 0
    box = Scene(boxes=[Aabb([0.2, -0.05, -0.1], [0.3, 0.05, 0.1])])
    hit, free = np.array([0.0, 0.0]), np.array([np.pi / 2, 0.0])
    for iters in (1, 2000):
        prm = PlanParams(width=8, max_iterations=iters)
        with pytest.raises(PlanSetupError, match="start is in collision"):
            plan(PlanProblem(m, box, None, hit, free, prm))
        with pytest.raises(PlanSetupError, match="goal is in collision"):
            plan(PlanProblem(m, box, None, free, hit, prm))
        with pytest.raises(PlanSetupError, match="start is in collision"):
            plan(PlanProblem(m, box, None, hit, hit + np.array([0.0, 0.3]), prm))
    # one team, valid endpoints: the query ends (IterLimit or solved), no hang
    r = plan(PlanProblem(m, box, None, free, np.array([2.5, 0.3]), PlanParams(width=8, max_iterations=1)))
    assert r.status in ("IterLimit", "Solved")
