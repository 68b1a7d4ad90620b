"""Clustered broad-phase collision checking (cprrtc_validate_broadphase and
the planner's cc_broadphase mode) against the reference's verdicts.

The broad phase changes which checks run and in what order, never the
verdict: every motion's valid/invalid outcome must equal the reference's
validate_waypoints (pure.py:646-699) except motions with a contact within
1e-5 m (the FP32 bar of test_gpu_parity.py).
"""

import numpy as np
import pytest

import fixtures as fx
from test_gpu_parity import CONTACT_TOL, _min_abs_clearance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2505_06791_b200 import kernels
    return kernels


def _motions(K, m, B, W, seed):
    qs = K.halton_batch(m, 2 * B, 1, seed)
    t = np.linspace(0.0, 1.0, W)[None, :, None]
    return qs[0::2][:, None, :] * (1 - t) + qs[1::2][:, None, :] * t


def test_broadphase_golden_verdicts(K, oracle):
    """The reference's golden validation sets: same verdicts, flag on and off."""
    k = fx.kats()
    keys = sorted({key[4:-4] for key in k if key.startswith("val_") and key.endswith("_wps")})
    compared = 0
    for key in keys:
        rname = "arm8_dense" if key.startswith("arm8_dense") else key.split("_")[0]
        m, sc = fx.robot(rname), fx.scene(key[len(rname) + 1:])
        res, wps_all = k[f"val_{key}_res"], k[f"val_{key}_wps"]
        for W in (8, 16):
            idx = [i for i in range(len(wps_all)) if res[2 * i][0] == W]
            if not idx:
                continue
            batch = np.stack([wps_all[i][:W] for i in idx])
            for flag in (0, 1):
                got = K.validate_batch(m, sc, batch, bool(flag), broadphase=True)
                for j, i in enumerate(idx):
                    v = bool(res[2 * i + flag][2])
                    if bool(got["valid"][j]) != v:
                        assert _min_abs_clearance(oracle, m, sc, batch[j]) < CONTACT_TOL, (key, i)
                    compared += 1
                    # first_bad = the lowest colliding waypoint
                    if not got["valid"][j] and flag == 0:
                        fb = got["first_bad"][j]
                        ok, *_ = oracle.validate_waypoints(batch[j][fb:fb + 1], m.packed, sc.packed(), False)
                        assert not ok or _min_abs_clearance(oracle, m, sc, batch[j][fb:fb + 1]) < CONTACT_TOL
    assert compared > 400


@pytest.mark.parametrize("scene", ["shelf_x11", "shelf_x111", "lattice75", "rand10_s4", "table"])
@pytest.mark.parametrize("robot", ["arm7", "arm8_dense"])
def test_broadphase_matches_lockstep(K, oracle, robot, scene):
    """Random motions through dense scenes: broad-phase verdicts equal the
    lockstep kernel's (itself pinned to the reference) and the oracle's."""
    m, sc = fx.robot(robot), fx.scene(scene)
    wps = _motions(K, m, 512, 16, 777)
    ref = K.validate_batch(m, sc, wps, False)
    for flag in (False, True):
        got = K.validate_batch(m, sc, wps, flag, broadphase=True)
        diff = np.nonzero(got["valid"] != ref["valid"])[0]
        for j in diff:
            assert _min_abs_clearance(oracle, m, sc, wps[j]) < CONTACT_TOL, (robot, scene, j)
        assert len(diff) <= 2
    # oracle spot check on a subset
    for j in range(0, 512, 37):
        v, *_ = oracle.validate_waypoints(wps[j], m.packed, sc.packed(), False)
        if v != bool(got["valid"][j]):
            assert _min_abs_clearance(oracle, m, sc, wps[j]) < CONTACT_TOL
    if scene.startswith("shelf_x"):
        # the point of the broad phase: far fewer checks than the lockstep order
        off = K.validate_batch(m, sc, wps, False, broadphase=True)
        assert off["performed"].sum() < 0.25 * ref["performed"].sum()


def test_broadphase_planner_paths(oracle):
    """Planning through the 999-box shelf in both check orders (the clustered
    broad phase and the reference's lockstep order): each must solve, over
    three seeds, and every path re-validates in FP64 (dense motions
    collision-free, on the manifold)."""
    from test_gpu_planner import _check_path
    from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanProblem, plan
    p = next(x for x in fx.plans() if x["id"] == "shelf_plane55_800")
    m, sp = fx.robot(p["robot"]), fx.spec(p["spec"])
    sc = fx.scene("shelf_x111")
    kw = dict(p["params"])
    kw["max_iterations"] = 200_000
    for bp in (1, 0):
        for seed in range(3):
            kw["seed_offset"] = seed * 10_000
            prob = PlanProblem(m, sc, sp, np.array(p["start"]), np.array(p["goal"]), PlanParams(**kw))
            res = plan(prob, DeviceOptions(cc_broadphase=bp))
            assert res.solved, (bp, seed, res.status)
            _check_path(oracle, prob, res)
