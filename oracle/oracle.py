"""ctypes front end of the C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
bench's CPU-baseline legs as the checker.  The product package never imports
this module.  Functions take the packed objects of either this repo's data
model or the reference's (duck-typed attribute access) and return numpy
arrays in the reference's shapes.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class _Robot(C.Structure):
    _fields_ = [("n", C.c_int), ("jtypes", _ip), ("axes", _dp), ("origin_r", _dp),
                ("origin_p", _dp), ("lo", _dp), ("hi", _dp), ("ns", C.c_int),
                ("sphere_link", _ip), ("sphere_local", _dp), ("sphere_radius", _dp),
                ("np", C.c_int), ("pairs", _ip), ("ee", C.c_int)]


class _Scene(C.Structure):
    _fields_ = [("nb", C.c_int), ("box_min", _dp), ("box_max", _dp), ("ne", C.c_int),
                ("sph_center", _dp), ("sph_radius", _dp)]


class _Spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("anchor", C.c_double * 3), ("offset", C.c_double),
                ("b1", C.c_double * 3), ("b2", C.c_double * 3), ("has_orient", C.c_int),
                ("q_fixed", C.c_double * 4), ("r_fixed_t", C.c_double * 9),
                ("weight", C.c_double), ("tau_task", C.c_double)]


class _Params(C.Structure):
    _fields_ = [("step_size", C.c_double), ("width", C.c_int), ("alpha", C.c_double),
                ("proj_max_iters", C.c_int), ("lam", C.c_double), ("tau_task", C.c_double),
                ("tau_sm", C.c_double), ("max_iterations", C.c_int),
                ("time_budget_ms", C.c_double), ("connect_tolerance", C.c_double),
                ("projection_mode", C.c_int), ("flag_on", C.c_int),
                ("seed_offset", C.c_int64), ("deterministic", C.c_int),
                ("attempts", C.c_int), ("max_connect_segments", C.c_int)]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int), ("path_len", C.c_int), ("path", _dp),
                ("sources", _ip), ("stats", C.c_int64 * 9), ("wall_ms", C.c_double)]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_sphere_aabb_clearance.restype = C.c_double
        L.orc_sphere_aabb_clearance.argtypes = [C.c_double] * 10
        L.orc_sphere_sphere_clearance.restype = C.c_double
        L.orc_sphere_sphere_clearance.argtypes = [C.c_double] * 8
        L.orc_radical_inverse.restype = C.c_double
        L.orc_radical_inverse.argtypes = [C.c_int64, C.c_int]
        L.orc_np_sum.restype = C.c_double
        L.orc_np_sum.argtypes = [_dp, C.c_int]
        L.orc_halton.argtypes = [C.c_int, C.c_int64, C.c_int64, _dp, _dp, _dp]
        _LIB = L
    return _LIB


def _d(a):
    return a.ctypes.data_as(_dp)


class Handle:
    """Keeps the numpy buffers referenced by a ctypes struct alive."""

    def __init__(self, struct, keep):
        self.s = struct
        self.keep = keep


def robot(packed) -> Handle:
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)    # noqa: E731
    keep = dict(jt=i32(packed.jtypes), ax=f64(packed.axes), orr=f64(packed.origin_r),
                op=f64(packed.origin_p), lo=f64(packed.lo), hi=f64(packed.hi),
                sl=i32(packed.sphere_link), sc=f64(packed.sphere_local).reshape(-1),
                sr=f64(packed.sphere_radius), pr=i32(packed.pairs).reshape(-1))
    keep["sc"] = np.ascontiguousarray(keep["sc"]) if keep["sc"].size else np.zeros(3)
    keep["sr"] = keep["sr"] if keep["sr"].size else np.zeros(1)
    keep["sl"] = keep["sl"] if keep["sl"].size else np.zeros(1, np.int32)
    keep["pr"] = keep["pr"] if keep["pr"].size else np.zeros(2, np.int32)
    s = _Robot(len(keep["jt"]), keep["jt"].ctypes.data_as(_ip), _d(keep["ax"]), _d(keep["orr"]),
               _d(keep["op"]), _d(keep["lo"]), _d(keep["hi"]), int(np.asarray(packed.sphere_radius).size),
               keep["sl"].ctypes.data_as(_ip), _d(keep["sc"]), _d(keep["sr"]),
               int(np.asarray(packed.pairs).reshape(-1, 2).shape[0]), keep["pr"].ctypes.data_as(_ip),
               int(packed.ee_link))
    return Handle(s, keep)


def scene(packed) -> Handle:
    def arr(a, shape_last):
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        return a if a.size else np.zeros(shape_last)
    keep = dict(bmin=arr(packed.box_min, 3), bmax=arr(packed.box_max, 3),
                sc=arr(packed.sph_center, 3), sr=arr(packed.sph_radius, 1))
    nb = int(np.asarray(packed.box_min).reshape(-1, 3).shape[0])
    ne = int(np.asarray(packed.sph_radius).reshape(-1).shape[0])
    s = _Scene(nb, _d(keep["bmin"]), _d(keep["bmax"]), ne, _d(keep["sc"]), _d(keep["sr"]))
    return Handle(s, keep)


def spec(packed) -> Handle:
    s = _Spec()
    s.kind = int(packed.kind)
    s.anchor[:] = [float(v) for v in packed.anchor]
    s.offset = float(packed.offset)
    b = np.asarray(packed.basis, dtype=float).reshape(2, 3)
    s.b1[:] = b[0].tolist()
    s.b2[:] = b[1].tolist()
    s.has_orient = int(packed.has_orient)
    s.q_fixed[:] = [float(v) for v in packed.q_fixed]
    s.r_fixed_t[:] = [float(v) for v in packed.r_fixed_t]
    s.weight = float(packed.weight)
    s.tau_task = float(packed.tau_task)
    return Handle(s, {})


# --------------------------------------------------------------------------
# reference _kernels protocol, FP64
# --------------------------------------------------------------------------

def sphere_aabb_clearance(*a):
    return lib().orc_sphere_aabb_clearance(*[float(v) for v in a])


def sphere_sphere_clearance(*a):
    return lib().orc_sphere_sphere_clearance(*[float(v) for v in a])


def frames(packed_robot, q):
    h = robot(packed_robot)
    q = np.ascontiguousarray(q, dtype=float)
    out = np.empty((h.s.n, 12))
    lib().orc_frames(C.byref(h.s), _d(q), _d(out))
    return out


def world_spheres(packed_robot, q):
    h = robot(packed_robot)
    q = np.ascontiguousarray(q, dtype=float)
    out = np.empty((h.s.ns, 4))
    lib().orc_world_spheres(C.byref(h.s), _d(q), _d(out) if h.s.ns else _d(np.empty(4)))
    return out


def ee_pose(packed_robot, q):
    h = robot(packed_robot)
    q = np.ascontiguousarray(q, dtype=float)
    out = np.empty(7)
    lib().orc_ee_pose(C.byref(h.s), _d(q), _d(out))
    return out


def task_error_at(packed_spec, pose7):
    h = spec(packed_spec)
    p = np.ascontiguousarray(pose7, dtype=float)
    e = np.empty(5)
    m = lib().orc_task_error_at(C.byref(h.s), _d(p), _d(e))
    return e[:m].copy()


def task_err_jac(packed_spec, packed_robot, q):
    hs, hr = spec(packed_spec), robot(packed_robot)
    q = np.ascontiguousarray(q, dtype=float)
    e = np.empty(5)
    J = np.empty(5 * hr.s.n)
    m = lib().orc_task_err_jac(C.byref(hs.s), C.byref(hr.s), _d(q), _d(e), _d(J))
    return e[:m].copy(), J[:m * hr.s.n].reshape(m, hr.s.n).copy()


def damped_step(jac, e, lam):
    """Returns the step, or None when J J^T + lam^2 I is not SPD."""
    jac = np.ascontiguousarray(np.atleast_2d(jac), dtype=float)
    e = np.ascontiguousarray(e, dtype=float)
    m, n = jac.shape
    out = np.empty(n)
    ok = lib().orc_damped_step(m, n, _d(jac), _d(e), C.c_double(lam), _d(out))
    return out if ok else None


def project_segment(wps, packed_robot, packed_spec, tau_task, tau_sm, alpha, lam,
                    max_iters, mode, collect_trace=False):
    hr, hs = robot(packed_robot), spec(packed_spec)
    wps = np.ascontiguousarray(wps, dtype=float)
    w, n = wps.shape
    xi = np.empty_like(wps)
    iters, prog, tlen = C.c_int(), C.c_int(), C.c_int()
    if collect_trace and mode != 2:
        txi = np.empty((max_iters, w, n))
        tprog = np.empty(max_iters, dtype=np.int32)
        ok = lib().orc_project_segment(C.byref(hr.s), C.byref(hs.s), w, _d(wps),
                                       C.c_double(tau_task), C.c_double(tau_sm),
                                       C.c_double(alpha), C.c_double(lam), max_iters, mode,
                                       _d(xi), C.byref(iters), C.byref(prog), _d(txi),
                                       tprog.ctypes.data_as(_ip), C.byref(tlen))
        trace = [(k + 1, int(tprog[k]), txi[k].copy()) for k in range(tlen.value)]
    else:
        ok = lib().orc_project_segment(C.byref(hr.s), C.byref(hs.s), w, _d(wps),
                                       C.c_double(tau_task), C.c_double(tau_sm),
                                       C.c_double(alpha), C.c_double(lam), max_iters, mode,
                                       _d(xi), C.byref(iters), C.byref(prog), None, None, None)
        trace = None
    return bool(ok), xi, iters.value, prog.value, trace


def validate_waypoints(wps, packed_robot, packed_scene, flag_on):
    hr, hc = robot(packed_robot), scene(packed_scene)
    wps = np.ascontiguousarray(wps, dtype=float)
    perf, poss, fb = C.c_int64(), C.c_int64(), C.c_int()
    ok = lib().orc_validate_waypoints(C.byref(hr.s), C.byref(hc.s), wps.shape[0], _d(wps),
                                      int(bool(flag_on)), C.byref(perf), C.byref(poss), C.byref(fb))
    return bool(ok), perf.value, poss.value, fb.value


def radical_inverse(index, base):
    return lib().orc_radical_inverse(int(index), int(base))


def halton(n, index, seed_offset, lo, hi):
    lo = np.ascontiguousarray(lo, dtype=float)
    hi = np.ascontiguousarray(hi, dtype=float)
    out = np.empty(n)
    lib().orc_halton(n, int(index), int(seed_offset), _d(lo), _d(hi), _d(out))
    return out


def nearest(nodes, q):
    nodes = np.ascontiguousarray(nodes, dtype=float)
    q = np.ascontiguousarray(q, dtype=float)
    return lib().orc_nearest(nodes.shape[0], nodes.shape[1], _d(nodes), _d(q))


def np_sum(a):
    a = np.ascontiguousarray(a, dtype=float)
    return lib().orc_np_sum(_d(a), a.size)


_STATUS = {0: "Solved", 1: "TimedOut", 2: "IterLimit"}
_SETUP = {-1: "start violates joint limits", -2: "start is off the constraint manifold",
          -3: "start is in collision", -4: "goal violates joint limits",
          -5: "goal is off the constraint manifold", -6: "goal is in collision"}
_SRC = {0: "start", 1: "junction", 2: "goal"}
STAT_KEYS = ("iterations", "extensions_attempted", "extensions_added",
             "projection_failures", "collision_rejections", "cc_performed",
             "cc_possible", "nodes_start", "nodes_goal")


def plan(packed_robot, packed_scene, packed_spec, start, goal, *, step_size=0.5,
         width=32, alpha=0.1, proj_max_iters=128, lam=1e-3, tau_task=None, tau_sm=None,
         max_iterations=10_000, time_budget_ms=10_000.0, connect_tolerance=None,
         projection_mode="parallel", flag_mode="on", seed_offset=0, deterministic=False,
         attempts=1, max_connect_segments=256):
    """The reference planner (planner.py:430-485) restated in C, FP64.

    ``packed_spec`` None means unconstrained (tau = inf).  Returns a dict with
    status, path (list of arrays), edge_sources, stats and wall_ms, or raises
    ValueError(<reference PlanSetupError message>) on a bad start/goal.
    """
    hr, hc = robot(packed_robot), scene(packed_scene)
    if packed_spec is None:
        s = _Spec()
        s.kind = 0
        s.anchor[:] = [0.0, 0.0, 1.0]
        s.q_fixed[:] = [1.0, 0.0, 0.0, 0.0]
        s.r_fixed_t[:] = [1, 0, 0, 0, 1, 0, 0, 0, 1]
        s.weight = 0.5
        s.tau_task = math.inf
        hs = Handle(s, {})
    else:
        hs = spec(packed_spec)
    modes = {"parallel": 0, "literal-gap": 1, "naive": 2}
    p = _Params(float(step_size), int(width), float(alpha), int(proj_max_iters), float(lam),
                math.nan if tau_task is None else float(tau_task),
                math.nan if tau_sm is None else float(tau_sm), int(max_iterations),
                float(time_budget_ms),
                math.nan if connect_tolerance is None else float(connect_tolerance),
                modes[projection_mode], int(flag_mode == "on"), int(seed_offset),
                int(bool(deterministic)), int(attempts), int(max_connect_segments))
    start = np.ascontiguousarray(start, dtype=float)
    goal = np.ascontiguousarray(goal, dtype=float)
    res = _Result()
    lib().orc_plan(C.byref(hr.s), C.byref(hc.s), C.byref(hs.s), C.byref(p), _d(start),
                   _d(goal), C.byref(res))
    try:
        if res.status < 0:
            raise ValueError(_SETUP[res.status])
        n = hr.s.n
        path = None
        sources = None
        if res.status == 0:
            arr = np.ctypeslib.as_array(res.path, shape=(res.path_len * n,)).reshape(res.path_len, n)
            path = [row.copy() for row in arr]
            sources = [_SRC[int(res.sources[k])] for k in range(res.path_len - 1)]
        return {"status": _STATUS[res.status], "path": path, "edge_sources": sources,
                "stats": dict(zip(STAT_KEYS, [int(v) for v in res.stats])),
                "wall_ms": res.wall_ms}
    finally:
        lib().orc_result_free(C.byref(res))
