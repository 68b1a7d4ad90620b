"""ctypes binding of libcprrtc.so (include/cprrtc.h).

The library is built in-tree (``csrc/Makefile`` -> ``libcprrtc.so`` next to
this file).  There is no CPU fallback: every device-backed function raises
``DeviceError`` when the library, the CUDA driver or the GPU is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DeviceError, SingularSystemError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcprrtc.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)

EXPORTS = (
    "cprrtc_abi_version", "cprrtc_last_error", "cprrtc_device_count", "cprrtc_codegen",
    "cprrtc_precompile", "cprrtc_device_source", "cprrtc_ctx_create", "cprrtc_ctx_destroy",
    "cprrtc_set_scene", "cprrtc_set_constraint", "cprrtc_prepare", "cprrtc_launch_count",
    "cprrtc_last_timing", "cprrtc_fk", "cprrtc_task_err_jac", "cprrtc_task_error_at",
    "cprrtc_project_config", "cprrtc_check_config", "cprrtc_validate", "cprrtc_project",
    "cprrtc_nearest", "cprrtc_halton", "cprrtc_plan", "cprrtc_derive_edges",
    "cprrtc_clearance", "cprrtc_damped_step", "cprrtc_flush_l2", "cprrtc_nearest_trees", "cprrtc_step",
    "cprrtc_validate_broadphase", "cprrtc_plan_race", "cprrtc_plan_multi", "cprrtc_plan_flat",
    "cprrtc_plan_submit", "cprrtc_plan_wait", "cprrtc_elapsed_ms",
)
MAX_RACE = 8


class Robot(C.Structure):
    _fields_ = [("n", C.c_int), ("jtypes", _ip), ("axes", _dp), ("origin_r", _dp),
                ("origin_p", _dp), ("lo", _dp), ("hi", _dp), ("n_spheres", C.c_int),
                ("sphere_link", _ip), ("sphere_local", _dp), ("sphere_radius", _dp),
                ("n_pairs", C.c_int), ("pairs", _ip), ("ee_link", C.c_int)]


class SceneDesc(C.Structure):
    _fields_ = [("n_boxes", C.c_int), ("box_min", _dp), ("box_max", _dp),
                ("n_spheres", C.c_int), ("sph_center", _dp), ("sph_radius", _dp)]


class ConstraintDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("anchor", C.c_double * 3), ("offset", C.c_double),
                ("basis", C.c_double * 6), ("has_orient", C.c_int),
                ("q_fixed", C.c_double * 4), ("r_fixed_t", C.c_double * 9),
                ("weight", C.c_double), ("tau_task", C.c_double)]


class Params(C.Structure):
    _fields_ = [("step_size", C.c_double), ("width", C.c_int), ("alpha", C.c_double),
                ("proj_max_iters", C.c_int), ("lam", C.c_double), ("tau_task", C.c_double),
                ("tau_sm", C.c_double), ("max_iterations", C.c_int),
                ("time_budget_ms", C.c_double), ("connect_tolerance", C.c_double),
                ("projection_mode", C.c_int), ("flag_on", C.c_int), ("deterministic", C.c_int),
                ("max_connect_segments", C.c_int), ("cc_margin", C.c_double),
                ("teams", C.c_int), ("tree_capacity", C.c_int), ("path_capacity", C.c_int),
                ("cc_broadphase", C.c_int)]


ST_COUNT = 12


class Result(C.Structure):
    _fields_ = [("status", C.c_int), ("setup_code", C.c_int), ("path_len", C.c_int),
                ("nodes_start", C.c_int), ("nodes_goal", C.c_int), ("device_ms", C.c_double),
                ("stats", C.c_uint64 * ST_COUNT)]


_lock = threading.Lock()
_LIB = None


def load():
    """Load libcprrtc.so (raises DeviceError if it was not built)."""
    global _LIB
    with _lock:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (make -C paper_2505_06791_b200/csrc); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            L.cprrtc_last_error.restype = C.c_char_p
            L.cprrtc_launch_count.restype = C.c_int64
            L.cprrtc_launch_count.argtypes = [C.c_void_p]
            L.cprrtc_flush_l2.argtypes = [C.c_void_p, C.c_size_t]
            for name in EXPORTS:
                if name not in ("cprrtc_last_error", "cprrtc_launch_count", "cprrtc_abi_version"):
                    getattr(L, name).restype = C.c_int
            _LIB = L
    return _LIB


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = load().cprrtc_last_error().decode(errors="replace")
    if rc == -1:
        raise ValueError(msg or what)
    if rc == -5:
        raise SingularSystemError(msg)
    raise DeviceError(f"{what}: {msg}" if what else msg)


def ptr(a, kind=_dp):
    return a.ctypes.data_as(kind) if a is not None else None


class RobotHandle:
    """A cprrtc_robot struct plus the arrays it points into."""

    def __init__(self, packed):
        f = lambda a, shape=None: np.ascontiguousarray(a, dtype=np.float64).reshape(-1)  # noqa: E731
        i = lambda a: np.ascontiguousarray(a, dtype=np.int32).reshape(-1)                # noqa: E731
        self.keep = dict(jt=i(packed.jtypes), ax=f(packed.axes), orr=f(packed.origin_r),
                         op=f(packed.origin_p), lo=f(packed.lo), hi=f(packed.hi),
                         sl=i(packed.sphere_link), sc=f(packed.sphere_local),
                         sr=f(packed.sphere_radius), pr=i(packed.pairs))
        for key, dt in (("sl", np.int32), ("sc", np.float64), ("sr", np.float64), ("pr", np.int32)):
            if self.keep[key].size == 0:
                self.keep[key] = np.zeros(4, dtype=dt)
        k = self.keep
        self.n = int(k["jt"].size)
        self.S = int(np.asarray(packed.sphere_radius).size)
        self.P = int(np.asarray(packed.pairs).reshape(-1, 2).shape[0])
        self.s = Robot(self.n, ptr(k["jt"], _ip), ptr(k["ax"]), ptr(k["orr"]), ptr(k["op"]),
                       ptr(k["lo"]), ptr(k["hi"]), self.S, ptr(k["sl"], _ip), ptr(k["sc"]),
                       ptr(k["sr"]), self.P, ptr(k["pr"], _ip), int(packed.ee_link))


class SceneHandle:
    def __init__(self, packed):
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64).reshape(-1)  # noqa: E731
        self.keep = [f(packed.box_min), f(packed.box_max), f(packed.sph_center), f(packed.sph_radius)]
        self.keep = [a if a.size else np.zeros(4) for a in self.keep]
        nb = int(np.asarray(packed.box_min).reshape(-1, 3).shape[0])
        ne = int(np.asarray(packed.sph_radius).reshape(-1).shape[0])
        self.s = SceneDesc(nb, ptr(self.keep[0]), ptr(self.keep[1]), ne, ptr(self.keep[2]),
                           ptr(self.keep[3]))


def constraint_desc(packed) -> ConstraintDesc:
    d = ConstraintDesc()
    d.kind = int(packed.kind)
    d.anchor[:] = [float(v) for v in np.asarray(packed.anchor).reshape(3)]
    d.offset = float(packed.offset)
    d.basis[:] = [float(v) for v in np.asarray(packed.basis).reshape(6)]
    d.has_orient = int(packed.has_orient)
    d.q_fixed[:] = [float(v) for v in np.asarray(packed.q_fixed).reshape(4)]
    d.r_fixed_t[:] = [float(v) for v in np.asarray(packed.r_fixed_t).reshape(9)]
    d.weight = float(packed.weight)
    d.tau_task = float(packed.tau_task)
    return d


def codegen(packed_robot) -> str:
    L = load()
    h = RobotHandle(packed_robot)
    need = C.c_size_t()
    check(L.cprrtc_codegen(C.byref(h.s), None, C.c_size_t(0), C.byref(need)), "codegen")
    buf = C.create_string_buffer(need.value)
    check(L.cprrtc_codegen(C.byref(h.s), buf, need, None), "codegen")
    return buf.value.decode()


def device_source(packed_robot, G=16, kind=0, orient=0, parity=0) -> str:
    L = load()
    h = RobotHandle(packed_robot)
    need = C.c_size_t()
    check(L.cprrtc_device_source(C.byref(h.s), G, kind, orient, parity, None, C.c_size_t(0),
                                 C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(L.cprrtc_device_source(C.byref(h.s), G, kind, orient, parity, buf, need, None))
    return buf.value.decode()


def precompile(packed_robot, G=16, kind=0, orient=0, parity=0) -> str:
    L = load()
    h = RobotHandle(packed_robot)
    buf = C.create_string_buffer(4096)
    check(L.cprrtc_precompile(C.byref(h.s), G, kind, orient, parity, buf, C.c_size_t(4096)),
          "precompile")
    return buf.value.decode()


def device_count() -> int:
    n = C.c_int(0)
    load().cprrtc_device_count(C.byref(n))
    return n.value
