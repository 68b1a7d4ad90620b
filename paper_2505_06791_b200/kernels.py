"""Device-backed kernel layer: contexts plus batched entry points.

Two faces:

* batched functions (``fk_batch``, ``validate_batch``, ``project_batch`` ...)
  used by the package's public API and the bench;
* the reference's kernel-backend protocol (``maniplan/_kernels/pure.py``:
  ``frames``, ``ee_pose``, ``world_spheres``, ``task_error_at``,
  ``task_err_jac``, ``damped_step``, ``project_segment``,
  ``validate_waypoints``, the two clearances and the MODE_* constants), so a
  reference install can select this module as its backend
  (INTEGRATION.md).  Results follow the device arithmetic: FP32 on the
  planning path (FK, task error/Jacobian, projection, collision checks), FP64
  for the setup-type helpers (clearances, damped step, Halton, endpoint
  checks, single-configuration projection).

Every call runs on the GPU through libcprrtc.so; there is no host fallback.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import threading

import numpy as np

from . import _lib
from .errors import DeviceError, SingularSystemError

name = "b200"
MODE_PARALLEL = 0
MODE_LITERAL_GAP = 1
MODE_SEQUENTIAL = 2

_dp, _ip, _lp = _lib._dp, _lib._ip, _lib._lp


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def _digest(*arrays) -> str:
    h = hashlib.sha1()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def robot_key(packed) -> str:
    return _digest(packed.jtypes, packed.axes, packed.origin_r, packed.origin_p, packed.lo,
                   packed.hi, packed.sphere_link, packed.sphere_local, packed.sphere_radius,
                   packed.pairs, np.array([packed.ee_link]))


def scene_key(packed) -> str:
    return _digest(packed.box_min, packed.box_max, packed.sph_center, packed.sph_radius)


def spec_key(packed) -> str:
    if packed is None:
        return "none"
    return _digest(np.array([packed.kind, packed.has_orient]), packed.anchor,
                   np.array([packed.offset, packed.weight, packed.tau_task]), packed.basis,
                   packed.q_fixed, packed.r_fixed_t)


class Context:
    """One libcprrtc context: a robot on one GPU plus its current scene and
    constraint (re-uploaded only when they change)."""

    def __init__(self, packed_robot, device: int = 0):
        L = _lib.load()
        self.robot = _lib.RobotHandle(packed_robot)
        self.n = self.robot.n
        self.S = self.robot.S
        self.P = self.robot.P
        self.device = device
        h = C.c_void_p()
        _lib.check(L.cprrtc_ctx_create(device, C.byref(self.robot.s), C.byref(h)), "context")
        self.h = h
        self.L = L
        self._scene = None
        self._spec = "none"
        self._scene_obj = None
        self._spec_obj = None
        self.kind = 0
        self.m = 1
        self.lock = threading.RLock()
        self._prepared = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.L.cprrtc_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- state -----------------------------------------------------------
    def set_scene(self, packed_scene):
        if packed_scene is self._scene_obj:
            return
        k = scene_key(packed_scene)
        self._scene_obj = packed_scene      # kept alive: identity stays valid
        if k != self._scene:
            sh = _lib.SceneHandle(packed_scene)
            _lib.check(self.L.cprrtc_set_scene(self.h, C.byref(sh.s)), "set_scene")
            self._scene = k
            self.nb = sh.s.n_boxes
            self.ne = sh.s.n_spheres

    def set_spec(self, packed_spec):
        if packed_spec is self._spec_obj and packed_spec is not None:
            return
        k = spec_key(packed_spec)
        self._spec_obj = packed_spec
        if k != self._spec:
            if packed_spec is None:
                _lib.check(self.L.cprrtc_set_constraint(self.h, None), "set_constraint")
                self.m = 1
            else:
                d = _lib.constraint_desc(packed_spec)
                _lib.check(self.L.cprrtc_set_constraint(self.h, C.byref(d)), "set_constraint")
                self.m = (1 if packed_spec.kind == 0 else 2) + (3 if packed_spec.has_orient else 0)
            self._spec = k

    def prepare(self, width: int):
        key = (self._spec, width)
        if key == self._prepared:      # module already loaded for this constraint kind / width
            return
        _lib.check(self.L.cprrtc_prepare(self.h, int(width)), "prepare")
        self._prepared = key

    @property
    def launches(self) -> int:
        return int(self.L.cprrtc_launch_count(self.h))

    def flush_l2(self, nbytes: int = 256 << 20):
        _lib.check(self.L.cprrtc_flush_l2(self.h, int(nbytes)), "flush_l2")

    def last_timing(self):
        a, b = C.c_double(), C.c_double()
        self.L.cprrtc_last_timing(self.h, C.byref(a), C.byref(b))
        return a.value, b.value


_CTX: dict = {}
_CTX_LOCK = threading.Lock()


_BY_ID: dict = {}


def context(model_or_packed, device: int = 0, slot: int = 0) -> Context:
    """The (robot, device, thread) context; ``slot`` > 0 gives further
    independent contexts on the same device (e.g. several racers on one GPU)."""
    packed = getattr(model_or_packed, "packed", model_or_packed)
    tid = threading.get_ident()
    hit = _BY_ID.get((id(packed), device, tid, slot))
    if hit is not None and hit[0] is packed:
        return hit[1]
    key = (robot_key(packed), device, tid, slot)
    with _CTX_LOCK:
        ctx = _CTX.get(key)
        if ctx is None:
            ctx = Context(packed, device)
            _CTX[key] = ctx
        _BY_ID[(id(packed), device, tid, slot)] = (packed, ctx)   # strong ref: ids stay unique
    return ctx


def _packed_spec(spec):
    if spec is None:
        return None
    return getattr(spec, "packed", spec)


def _packed_scene(scene):
    return scene.packed() if callable(getattr(scene, "packed", None)) else scene


# ---------------------------------------------------------------------------
# batched entry points
# ---------------------------------------------------------------------------

def fk_batch(model, q, fp64: bool = False, device: int = 0) -> dict:
    ctx = context(model, device)
    q = _f64(q)
    B = q.shape[0]
    n, S = ctx.n, ctx.S
    out = dict(frames=np.empty((B, n, 12)), axes=np.empty((B, n, 3)),
               origins=np.empty((B, n, 3)), ee=np.empty((B, 7)),
               spheres=np.empty((B, S, 4)))
    with ctx.lock:
        _lib.check(ctx.L.cprrtc_fk(ctx.h, B, _lib.ptr(q), int(fp64), _lib.ptr(out["frames"]),
                                   _lib.ptr(out["axes"]), _lib.ptr(out["origins"]),
                                   _lib.ptr(out["ee"]), _lib.ptr(out["spheres"]) if S else None),
                   "fk")
    return out


def task_err_jac_batch(model, spec, q, fp64: bool = False, device: int = 0):
    ctx = context(model, device)
    q = _f64(q)
    B = q.shape[0]
    with ctx.lock:
        ctx.set_spec(_packed_spec(spec))
        m = ctx.m
        e = np.empty((B, m))
        J = np.empty((B, m, ctx.n))
        _lib.check(ctx.L.cprrtc_task_err_jac(ctx.h, B, _lib.ptr(q), int(fp64), _lib.ptr(e),
                                             _lib.ptr(J)), "task_err_jac")
    return e, J


def task_error_at(packed_spec, pose7):
    """FP64 task error at a pose; needs no robot (any cached context works)."""
    pose = _f64(pose7).reshape(-1, 7)
    ctx = _pose_context()
    with ctx.lock:
        ctx.set_spec(packed_spec)
        e = np.empty((pose.shape[0], ctx.m))
        _lib.check(ctx.L.cprrtc_task_error_at(ctx.h, pose.shape[0], _lib.ptr(pose), _lib.ptr(e)),
                   "task_error_at")
    return e[0] if np.ndim(pose7) == 1 else e


_POSE_STUB = None


def _pose_context() -> Context:
    """A private context (1-joint stub robot, this thread) for the robot-free
    pose helpers: it never shares constraint state with a planning context."""
    global _POSE_STUB
    if _POSE_STUB is None:
        from types import SimpleNamespace
        _POSE_STUB = SimpleNamespace(
            jtypes=np.zeros(1, np.int32), axes=np.array([[0, 0, 1.0]]),
            origin_r=np.eye(3).reshape(1, 9), origin_p=np.zeros((1, 3)),
            lo=np.array([-1.0]), hi=np.array([1.0]), sphere_link=np.zeros(0, np.int32),
            sphere_local=np.zeros((0, 3)), sphere_radius=np.zeros(0),
            pairs=np.zeros((0, 2), np.int32), ee_link=0)
    return context(_POSE_STUB, 0, slot=-1)


def damped_step(jac, e, lam, device: int = 0):
    jac = _f64(np.atleast_2d(jac))
    m, n = jac.shape
    e = _f64(e).reshape(m)
    out = np.empty(n)
    ok = np.zeros(1, np.int32)
    _lib.check(_lib.load().cprrtc_damped_step(device, 1, m, n, _lib.ptr(jac), _lib.ptr(e),
                                              C.c_double(lam), _lib.ptr(out), _lib.ptr(ok, _ip)),
               "damped_step")
    if not ok[0]:
        raise SingularSystemError("J J^T is singular; use lam > 0 for a damped solve")
    return out


def damped_step_batch(jac, e, lam, device: int = 0):
    jac = _f64(jac)
    B, m, n = jac.shape
    e = _f64(e).reshape(B, m)
    out = np.empty((B, n))
    ok = np.zeros(B, np.int32)
    _lib.check(_lib.load().cprrtc_damped_step(device, B, m, n, _lib.ptr(jac), _lib.ptr(e),
                                              C.c_double(lam), _lib.ptr(out), _lib.ptr(ok, _ip)),
               "damped_step")
    return out, ok.astype(bool)


def clearance_batch(spheres, others, kind: str = "box", device: int = 0):
    """FP64 clearances: spheres (B,4) [x,y,z,r] vs boxes (B,6) [lo,hi] or
    spheres (B,4)."""
    a = _f64(spheres).reshape(-1, 4)
    b = _f64(others).reshape(a.shape[0], 6 if kind == "box" else 4)
    out = np.empty(a.shape[0])
    _lib.check(_lib.load().cprrtc_clearance(device, a.shape[0], 0 if kind == "box" else 1,
                                            _lib.ptr(a), _lib.ptr(b), _lib.ptr(out)), "clearance")
    return out


def validate_batch(model, scene, wps, flag_on: bool = True, margin: float = 0.0, device: int = 0,
                   broadphase: bool = False):
    """B motions (B, W, n) -> dict(valid, first_bad, performed, possible, gpu_checks).

    broadphase=False: the reference's lockstep order with its exact counters;
    True: the clustered broad phase (same verdicts, its own counters)."""
    ctx = context(model, device)
    wps = _f64(wps)
    if wps.ndim == 2:
        wps = wps[None]
    B, W, n = wps.shape
    if n != ctx.n:
        raise ValueError("waypoint dimension does not match the model")
    r = dict(valid=np.empty(B, np.int32), first_bad=np.empty(B, np.int32),
             performed=np.empty(B, np.int64), possible=np.empty(B, np.int64),
             gpu_checks=np.empty(B, np.int64))
    with ctx.lock:
        ctx.set_scene(_packed_scene(scene))
        fn = ctx.L.cprrtc_validate_broadphase if broadphase else ctx.L.cprrtc_validate
        _lib.check(fn(
            ctx.h, B, W, _lib.ptr(wps), int(bool(flag_on)), C.c_double(margin),
            _lib.ptr(r["valid"], _ip), _lib.ptr(r["first_bad"], _ip), _lib.ptr(r["performed"], _lp),
            _lib.ptr(r["possible"], _lp), _lib.ptr(r["gpu_checks"], _lp)), "validate")
        r["kernel_ms"] = ctx.last_timing()[1]
    r["valid"] = r["valid"].astype(bool)
    return r


def project_batch(model, spec, wps, tau_task, tau_sm, alpha=0.1, lam=1e-3, max_iters=128,
                  mode=0, collect_trace=False, device: int = 0):
    """B segments (B, W, n); tau_sm scalar, (B,) or None (auto)."""
    ctx = context(model, device)
    wps = _f64(wps)
    if wps.ndim == 2:
        wps = wps[None]
    B, W, n = wps.shape
    tsm = None
    if tau_sm is not None:
        tsm = _f64(np.broadcast_to(np.asarray(tau_sm, dtype=float), (B,)))
    xi = np.empty_like(wps)
    ok = np.empty(B, np.int32)
    iters = np.empty(B, np.int32)
    prog = np.empty(B, np.int32)
    trace = tprog = None
    if collect_trace:
        trace = np.empty((B, max_iters, W, n))
        tprog = np.empty((B, max_iters), np.int32)
    with ctx.lock:
        ctx.set_spec(_packed_spec(spec))
        _lib.check(ctx.L.cprrtc_project(
            ctx.h, B, W, _lib.ptr(wps), _lib.ptr(tsm), C.c_double(tau_task), C.c_double(alpha),
            C.c_double(lam), int(max_iters), int(mode), _lib.ptr(xi), _lib.ptr(ok, _ip),
            _lib.ptr(iters, _ip), _lib.ptr(prog, _ip), _lib.ptr(trace),
            _lib.ptr(tprog, _ip) if tprog is not None else None), "project")
    return dict(ok=ok.astype(bool), xi=xi, iters=iters, prog=prog, trace=trace, trace_prog=tprog)


def nearest_batch(model, nodes, queries, device: int = 0):
    ctx = context(model, device)
    nodes = _f64(nodes)
    queries = _f64(queries).reshape(-1, nodes.shape[1])
    idx = np.empty(queries.shape[0], np.int32)
    with ctx.lock:
        _lib.check(ctx.L.cprrtc_nearest(ctx.h, nodes.shape[0], _lib.ptr(nodes), queries.shape[0],
                                        _lib.ptr(queries), _lib.ptr(idx, _ip)), "nearest")
    return idx


def nearest_trees(model, nodes, queries, device: int = 0):
    """Query i scans tree i % T of nodes (T, N, n); returns (idx, kernel_ms)."""
    ctx = context(model, device)
    nodes = _f64(nodes)
    T, N, n = nodes.shape
    queries = _f64(queries).reshape(-1, n)
    idx = np.empty(queries.shape[0], np.int32)
    with ctx.lock:
        _lib.check(ctx.L.cprrtc_nearest_trees(ctx.h, N, T, None, _lib.ptr(nodes), queries.shape[0],
                                              _lib.ptr(queries), _lib.ptr(idx, _ip)), "nearest")
        ms = ctx.last_timing()[1]
    return idx, ms


def halton_batch(model, count: int, first_index: int = 1, seed_offset: int = 0, limits=None,
                 device: int = 0):
    """``count`` Halton samples from index ``first_index`` (FP64, bit-exact)."""
    ctx = context(model, device)
    out = np.empty((int(count), ctx.n))
    lo = hi = None
    if limits is not None:
        limits = _f64(limits).reshape(ctx.n, 2)
        lo, hi = np.ascontiguousarray(limits[:, 0]), np.ascontiguousarray(limits[:, 1])
    with ctx.lock:
        _lib.check(ctx.L.cprrtc_halton(ctx.h, int(count), C.c_int64(first_index),
                                       C.c_int64(seed_offset), _lib.ptr(lo), _lib.ptr(hi),
                                       _lib.ptr(out)), "halton")
    return out


def project_config_batch(model, spec, q, tau, lam=1e-3, max_iters=128, device: int = 0):
    ctx = context(model, device)
    q = _f64(q).copy().reshape(-1, ctx.n)
    ok = np.empty(q.shape[0], np.int32)
    with ctx.lock:
        ctx.set_spec(_packed_spec(spec))
        _lib.check(ctx.L.cprrtc_project_config(ctx.h, q.shape[0], _lib.ptr(q), C.c_double(tau),
                                               C.c_double(lam), int(max_iters), _lib.ptr(ok, _ip)),
                   "project_config")
    return q, ok.astype(bool)


def check_config_batch(model, scene, spec, q, tau=None, device: int = 0):
    """0 ok, 1 limits, 2 off manifold, 3 collision (FP64, planner.py:416-427)."""
    ctx = context(model, device)
    q = _f64(q).reshape(-1, ctx.n)
    code = np.empty(q.shape[0], np.int32)
    ps = _packed_spec(spec)
    if tau is None:
        tau = math.inf if ps is None else float(ps.tau_task)
    with ctx.lock:
        ctx.set_scene(_packed_scene(scene))
        ctx.set_spec(ps)
        _lib.check(ctx.L.cprrtc_check_config(ctx.h, q.shape[0], _lib.ptr(q), C.c_double(tau),
                                             _lib.ptr(code, _ip)), "check_config")
    return code


# ---------------------------------------------------------------------------
# the reference kernel-backend protocol (maniplan/_kernels/pure.py)
# ---------------------------------------------------------------------------

def sphere_aabb_clearance(cx, cy, cz, r, lx, ly, lz, hx, hy, hz):
    return float(clearance_batch([[cx, cy, cz, r]], [[lx, ly, lz, hx, hy, hz]], "box")[0])


def sphere_sphere_clearance(ax, ay, az, ar, bx, by, bz, br):
    return float(clearance_batch([[ax, ay, az, ar]], [[bx, by, bz, br]], "sphere")[0])


def rot_from_quat(w, x, y, z):
    xx, yy, zz, xy, xz, yz = x * x, y * y, z * z, x * y, x * z, y * z
    wx, wy, wz = w * x, w * y, w * z
    return (1.0 - 2.0 * (yy + zz), 2.0 * (xy - wz), 2.0 * (xz + wy),
            2.0 * (xy + wz), 1.0 - 2.0 * (xx + zz), 2.0 * (yz - wx),
            2.0 * (xz - wy), 2.0 * (yz + wx), 1.0 - 2.0 * (xx + yy))


def frames(packed_robot, q):
    return fk_batch(packed_robot, _f64(q)[None])["frames"][0]


def ee_pose(packed_robot, q):
    return fk_batch(packed_robot, _f64(q)[None])["ee"][0]


def world_spheres(packed_robot, q):
    return fk_batch(packed_robot, _f64(q)[None])["spheres"][0]


def task_err_jac(packed_spec, packed_robot, q):
    e, J = task_err_jac_batch(packed_robot, packed_spec, _f64(q)[None])
    return e[0], J[0]


def project_segment(wps, packed_robot, packed_spec, tau_task, tau_sm, alpha, lam, max_iters,
                    mode, collect_trace=False):
    r = project_batch(packed_robot, packed_spec, _f64(wps)[None], tau_task, tau_sm, alpha, lam,
                      max_iters, mode, collect_trace and mode != MODE_SEQUENTIAL)
    trace = None
    if r["trace"] is not None:
        tp = r["trace_prog"][0]
        k = int((tp >= 0).sum())
        trace = [(i + 1, int(tp[i]), r["trace"][0, i].copy()) for i in range(k)]
    return bool(r["ok"][0]), r["xi"][0], int(r["iters"][0]), int(r["prog"][0]), trace


def validate_waypoints(wps, packed_robot, packed_scene, flag_on):
    r = validate_batch(packed_robot, packed_scene, _f64(wps)[None], flag_on)
    return (bool(r["valid"][0]), int(r["performed"][0]), int(r["possible"][0]),
            int(r["first_bad"][0]))


__all__ = [
    "name", "MODE_PARALLEL", "MODE_LITERAL_GAP", "MODE_SEQUENTIAL", "Context", "context",
    "fk_batch", "task_err_jac_batch", "task_error_at", "damped_step", "damped_step_batch",
    "clearance_batch", "validate_batch", "project_batch", "nearest_batch", "halton_batch",
    "project_config_batch", "check_config_batch", "sphere_aabb_clearance",
    "sphere_sphere_clearance", "rot_from_quat", "frames", "ee_pose", "world_spheres",
    "task_err_jac", "project_segment", "validate_waypoints", "DeviceError",
]
