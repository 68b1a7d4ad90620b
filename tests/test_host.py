"""Host-side logic that needs no GPU: data model, segment construction,
tree bookkeeping, path assembly and parameter validation."""

import numpy as np
import pytest

import fixtures as fx
from paper_2505_06791_b200.geometry import Aabb, Scene, Sphere, scene_contains
from paper_2505_06791_b200.planner import PlanParams, Tree, extract_path, steer
from paper_2505_06791_b200.projection import (MotionSegment, ProjectionParams,
                                              interpolate_segment, segment_gaps)


def test_interpolate_segment():
    seg = interpolate_segment([0.0, 0.0], [2.0, 2.0], 3)
    assert np.array_equal(seg.waypoints, [[0, 0], [1, 1], [2, 2]])
    a, b = np.array([0.1, 0.2, 0.3]), np.array([-0.7, 0.4, 1.1])
    seg = interpolate_segment(a, b, 7)
    assert np.array_equal(seg.start, a) and np.array_equal(seg.end, b)
    g = segment_gaps(seg)
    assert np.allclose(g, g[0], atol=1e-12)
    with pytest.raises(ValueError, match="width"):
        interpolate_segment([0.0], [1.0], 1)
    with pytest.raises(ValueError, match="same length"):
        interpolate_segment([0.0], [1.0, 2.0], 4)
    with pytest.raises(ValueError, match="W >= 2"):
        MotionSegment(np.zeros((1, 3)))


def test_interpolation_matches_reference_formula(oracle):
    rng = np.random.default_rng(1)
    for _ in range(50):
        a, b = rng.normal(size=7), rng.normal(size=7)
        W = int(rng.integers(2, 33))
        ref = np.array([a + (k / (W - 1)) * (b - a) for k in range(W)])
        ref[0], ref[-1] = a, b
        assert np.array_equal(interpolate_segment(a, b, W).waypoints, ref)


def test_params_validation():
    with pytest.raises(ValueError):
        ProjectionParams(alpha=0.0)
    with pytest.raises(ValueError):
        ProjectionParams(tau_sm=0.0)
    with pytest.raises(ValueError):
        PlanParams(step_size=0)
    with pytest.raises(ValueError):
        PlanParams(attempts=0)
    assert PlanParams(step_size=0.4).tolerance == pytest.approx(0.04)


def test_tree_and_path_assembly():
    t = Tree([0.0, 0.0], "start")
    a = t.add([1.0, 0.0], 0)
    b = t.add([1.0, 1.0], a)
    assert t.chain(b) == [0, 1, 2]
    with pytest.raises(IndexError):
        t.node(3)
    for i in range(200):
        t.add([float(i), 0.0], 0)
    assert len(t) == 203
    ts = Tree([0.0, 0.0], "start")
    ms = ts.add([1.0, 0.0], 0)
    tg = Tree([3.0, 0.0], "goal")
    mg = tg.add([1.0, 0.0], 0)
    path, src = extract_path(ts, tg, ms, mg)
    assert [tuple(p) for p in path] == [(0, 0), (1, 0), (3, 0)] and src == ("start", "goal")
    tg2 = Tree([3.0, 0.0], "goal")
    mg2 = tg2.add([1.02, 0.0], 0)
    path, src = extract_path(ts, tg2, ms, mg2)
    assert len(path) == 4 and src == ("start", "junction", "goal")


def test_steer():
    assert np.allclose(steer([0.0, 0.0], [3.0, 4.0], 1.0), [0.6, 0.8], atol=1e-15)
    t = np.array([0.3, -0.4])
    got = steer([0.0, 0.0], t, 1.0)
    assert np.array_equal(got, t) and got is not t


def test_scene_queries_and_q_checks():
    assert scene_contains(Scene(boxes=[Aabb([0, 0, 0], [1, 1, 1])]), [0.5, 0.5, 1.0])
    assert not scene_contains(Scene(spheres=[Sphere([0, 0, 0], 0.5)]), [0.5, 0.1, 0])
    with pytest.raises(ValueError):
        fx.robot("arm8").check_q(np.zeros(3))


def test_plan_race_argument_checks():
    """plan_race validates its racer list before touching a device."""
    import pytest
    from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan_race
    m = fx.robot("planar2")
    prob = PlanProblem(m, fx.scene("empty"), None, np.zeros(2), np.array([1.0, 0.5]), PlanParams())
    with pytest.raises(ValueError):
        plan_race(prob, devices=())
    with pytest.raises(ValueError):
        plan_race(prob, devices=tuple(range(9)))


def test_batch_arena_reused_only_without_live_views():
    """A result arena goes back to plan_many only when its BatchResult and
    every view a caller kept of its buffers (rows, codes, ...) are gone."""
    import gc
    from paper_2505_06791_b200 import planner as P
    B, pc, n = 3, 4, 2
    key = (B, pc, n)

    def result():
        a = P._arena(B, pc, n)
        a.offsets[:] = 0
        st = np.zeros((B, n))
        return a, P._batch_result(a, a.res, a.offsets, a.paths[:0], a.srcs[:0], st, st, 0.0, B, pc)

    P._TLS.arenas = {}
    a1, r1 = result()
    assert P._arena(B, pc, n) is not a1          # owned by a live result
    P._TLS.arenas = {key: [a1]}
    codes, rows = r1.codes, r1.rows
    del r1
    gc.collect()
    assert not a1.free()                         # views still alive
    assert P._arena(B, pc, n) is not a1
    P._TLS.arenas = {key: [a1]}
    del codes, rows
    gc.collect()
    assert a1.free()
    assert P._arena(B, pc, n) is a1
