"""Constrained bidirectional RRT-Connect on the B200.

Drop-in for ``maniplan/planner.py``: the same PlanParams / PlanProblem /
PlanResult / PlanStats types and the same ``plan(problem) -> PlanResult``
call, but the whole tree-extension loop -- sampling, nearest neighbour,
steering, parallel projection, FK + collision checking, greedy connect,
junction test and termination -- runs inside one persistent sm_100a kernel
(``csrc/device/cprrtc_device.cuh: cp_plan_kernel``).  Many teams extend the
two trees concurrently; sample i of the Halton stream (index i +
seed_offset, the reference's stream) extends the start tree when i is odd,
exactly like reference iteration i (planner.py:449-459).

Differences from the reference, all deliberate:
* FP32 device arithmetic with safety margins (tau_task x (1-1e-3) - 2e-6,
  tau_sm x (1-1e-5), robot spheres inflated by ``cc_margin`` = 1e-5 m), so
  every returned path re-validates in FP64.
* Extensions run concurrently, so a run is not bit-reproducible across
  launches; ``deterministic`` keeps its reference meaning (ignore the wall
  clock).  ``attempts`` is accepted; the device already evaluates hundreds of
  samples at once.
* ``stats.iterations`` counts samples drawn; ``cc_possible`` is the
  reference's count (every waypoint of every checked motion, row 0
  included, like validate_motion).  ``cc_performed`` follows the
  reference's lockstep accounting with ``DeviceOptions(cc_broadphase=0)``;
  with the clustered broad phase (the default whenever the scene has
  obstacles) it counts the sphere-primitive checks actually evaluated.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import sys
import threading
import time
import weakref
from contextlib import contextmanager
from collections.abc import Sequence
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib, kernels
from .constraints import ConstraintSpec, task_error, unconstrained
from .errors import PlanSetupError
from .geometry import Scene
from .kinematics import RobotModel, forward_kinematics
from .projection import MotionSegment, ProjectionParams

__all__ = [
    "Tree", "PlanParams", "PlanProblem", "PlanResult", "PlanStats", "PlanContext",
    "ExtendOutcome", "ConnectOutcome", "DeviceOptions", "nearest", "steer", "plan",
    "plan_batch", "extract_path", "derive_edge", "derive_path", "revalidate_path", "dense_path", "extend",
    "connect", "prepare", "plan_race", "plan_many", "BatchResult", "PlanStream",
]


class Tree:
    """Host-side append-only tree (API parity with maniplan.planner.Tree)."""

    def __init__(self, root, root_kind: str):
        root = np.asarray(root, dtype=float)
        self.root_kind = root_kind
        self._buf = np.empty((64, root.shape[0]))
        self._buf[0] = root
        self._len = 1
        self.parents = [0]

    def __len__(self):
        return self._len

    @property
    def nodes(self) -> np.ndarray:
        return self._buf[:self._len]

    def node(self, i: int) -> np.ndarray:
        if not 0 <= i < self._len:
            raise IndexError(f"node {i} out of range")
        return self._buf[i].copy()

    def add(self, q, parent: int) -> int:
        if not 0 <= parent < self._len:
            raise IndexError(f"parent {parent} out of range")
        if self._len == len(self._buf):
            self._buf = np.concatenate([self._buf, np.empty_like(self._buf)])
        self._buf[self._len] = np.asarray(q, dtype=float)
        self.parents.append(parent)
        self._len += 1
        return self._len - 1

    def chain(self, i: int) -> list:
        out = [i]
        while self.parents[i] != i:
            i = self.parents[i]
            out.append(i)
        return out[::-1]


@dataclass(frozen=True)
class PlanParams:
    step_size: float = 0.5
    width: int = 32
    projection: ProjectionParams = ProjectionParams()
    max_iterations: int = 10_000
    time_budget_ms: float = 10_000.0
    connect_tolerance: float | None = None
    projection_mode: str = "parallel"     # parallel | literal-gap | naive
    flag_mode: str = "on"
    seed_offset: int = 0
    deterministic: bool = False
    attempts: int = 1
    max_connect_segments: int = 256

    def __post_init__(self):
        if self.step_size <= 0 or self.width < 2:
            raise ValueError("step_size > 0 and width >= 2 required")
        if self.max_iterations < 1 or self.attempts < 1:
            raise ValueError("max_iterations and attempts must be >= 1")

    @property
    def tolerance(self) -> float:
        return self.connect_tolerance if self.connect_tolerance is not None else self.step_size / 10.0


@dataclass(frozen=True)
class DeviceOptions:
    """B200 knobs (no reference counterpart)."""

    device: int = 0
    teams: int = 0               # concurrent extension teams; 0 = automatic (single query: 192 two-warp
                                 # teams; batches: B + B/8, at least half the resident teams)
    cc_margin: float = 1e-5      # planner robot-sphere inflation (m)
    tree_capacity: int = 0       # nodes per tree; 0 = derived from the params
    path_capacity: int = 1024
    # planner collision checks through the clustered broad phase (same
    # verdicts; cc_performed then counts the checks evaluated): 1 on, 0 the
    # reference's lockstep order, -1 auto (on whenever the scene has obstacles)
    cc_broadphase: int = -1


@dataclass(frozen=True)
class PlanProblem:
    model: RobotModel
    scene: Scene
    spec: ConstraintSpec | None
    start: np.ndarray
    goal: np.ndarray
    params: PlanParams = PlanParams()
    name: str = ""

    def __post_init__(self):
        object.__setattr__(self, "start", self.model.check_q(self.start))
        object.__setattr__(self, "goal", self.model.check_q(self.goal))


@dataclass(slots=True)
class PlanStats:
    iterations: int = 0
    extensions_attempted: int = 0
    extensions_added: int = 0
    projection_failures: int = 0
    collision_rejections: int = 0
    cc_performed: int = 0
    cc_possible: int = 0
    wall_ms: float = 0.0
    nodes_start: int = 0
    nodes_goal: int = 0
    device_ms: float = 0.0        # query time on the device (globaltimer)
    # device work units (roofline accounting; no reference counterpart)
    stage1_evals: int = 0
    cc_fk_evals: int = 0
    nn_nodes: int = 0
    proj_iters: int = 0


@dataclass(frozen=True)
class PlanResult:
    status: str              # Solved | TimedOut | IterLimit (+ CapacityExceeded, Stopped; see _STATUS)
    path: tuple | None
    edge_sources: tuple | None
    stats: PlanStats
    dense: np.ndarray | None = field(default=None, compare=False)   # (E, W, n) on request

    @property
    def solved(self) -> bool:
        return self.status == "Solved"


@dataclass
class PlanContext:
    model: RobotModel
    scene: Scene
    spec: ConstraintSpec
    params: PlanParams
    stats: PlanStats = field(default_factory=PlanStats)
    options: DeviceOptions = DeviceOptions()

    @classmethod
    def from_problem(cls, problem: PlanProblem, options: DeviceOptions = DeviceOptions()):
        spec = problem.spec if problem.spec is not None else unconstrained()
        return cls(problem.model, problem.scene, spec, problem.params, options=options)


@dataclass(frozen=True)
class ExtendOutcome:
    status: str
    node: int | None = None
    reason: str | None = None

    @property
    def added(self) -> bool:
        return self.status == "Added"


@dataclass(frozen=True)
class ConnectOutcome:
    status: str
    node: int | None = None
    segments: int = 0

    @property
    def reached(self) -> bool:
        return self.status == "Reached"


_MODES = {"parallel": 0, "literal-gap": 1, "naive": 2}
# 3: a tree reached DeviceOptions.tree_capacity before a solution, the time
#    budget or max_iterations (no reference counterpart: its trees are
#    unbounded); 5: another racer solved the query (plan_race)
_STATUS = {0: "Solved", 1: "TimedOut", 2: "IterLimit", 3: "CapacityExceeded", 5: "Stopped"}
_SETUP = {1: "start violates joint limits", 2: "start is off the constraint manifold",
          3: "start is in collision", 4: "goal violates joint limits",
          5: "goal is off the constraint manifold", 6: "goal is in collision"}
_SRC = ("start", "junction", "goal")


def nearest(tree: Tree, q) -> int:
    """Index of the closest node, lowest index on ties (device scan)."""
    n = tree.nodes.shape[1]
    from types import SimpleNamespace
    # the scan is robot-independent apart from the dimension: a stub robot of
    # the right width selects the compiled module
    stub = _stub_robot(n)
    return int(kernels.nearest_batch(stub, tree.nodes, np.asarray(q, dtype=float)[None])[0])


_STUBS: dict = {}


def _stub_robot(n: int):
    from types import SimpleNamespace
    if n not in _STUBS:
        _STUBS[n] = SimpleNamespace(
            jtypes=np.zeros(n, np.int32), axes=np.tile([0.0, 0.0, 1.0], (n, 1)),
            origin_r=np.tile(np.eye(3).reshape(9), (n, 1)), origin_p=np.zeros((n, 3)),
            lo=np.full(n, -np.pi), hi=np.full(n, np.pi), sphere_link=np.zeros(0, np.int32),
            sphere_local=np.zeros((0, 3)), sphere_radius=np.zeros(0),
            pairs=np.zeros((0, 2), np.int32), ee_link=n - 1)
    return _STUBS[n]


def steer(q_near, q_rand, step: float):
    q_near = np.asarray(q_near, dtype=float)
    q_rand = np.asarray(q_rand, dtype=float)
    d = q_rand - q_near
    dist = float(np.sqrt((d * d).sum()))
    return q_rand.copy() if dist <= step else q_near + (step / dist) * d


_PRM_CACHE: dict = {}


def _params_struct(p: PlanParams, opt: DeviceOptions) -> _lib.Params:
    key = (id(p), id(opt))
    hit = _PRM_CACHE.get(key)
    if hit is not None and hit[0] is p and hit[1] is opt:
        return hit[2]
    prm = _make_params(p, opt)
    if len(_PRM_CACHE) > 4096:
        _PRM_CACHE.clear()
    _PRM_CACHE[key] = (p, opt, prm)
    return prm


def _make_params(p: PlanParams, opt: DeviceOptions) -> _lib.Params:
    pp = p.projection
    if p.projection_mode not in _MODES:
        raise ValueError(f"unknown projection mode {p.projection_mode!r}")
    if p.flag_mode not in ("on", "off"):
        raise ValueError(f"flag_mode must be 'on' or 'off', got {p.flag_mode!r}")
    return _lib.Params(
        step_size=float(p.step_size), width=int(p.width), alpha=float(pp.alpha),
        proj_max_iters=int(pp.max_iters), lam=float(pp.lam),
        tau_task=float(pp.tau_task) if pp.tau_task is not None else 0.0,
        tau_sm=float(pp.tau_sm) if pp.tau_sm is not None else 0.0,
        max_iterations=int(p.max_iterations), time_budget_ms=float(p.time_budget_ms),
        connect_tolerance=float(p.tolerance), projection_mode=_MODES[p.projection_mode],
        flag_on=int(p.flag_mode == "on"), deterministic=int(bool(p.deterministic)),
        max_connect_segments=int(p.max_connect_segments), cc_margin=float(opt.cc_margin),
        teams=int(opt.teams), tree_capacity=int(opt.tree_capacity),
        path_capacity=int(opt.path_capacity), cc_broadphase=int(opt.cc_broadphase))


@contextmanager
def _bound(problem_like, opt: DeviceOptions):
    """The problem's context with its lock held and its scene and constraint
    uploaded: the bind and every launch that depends on it run under one
    lock, so no other caller can swap the constraint in between."""
    ctx = kernels.context(problem_like.model, opt.device)
    with ctx.lock:
        ctx.set_scene(_scene_packed(problem_like.scene))
        ctx.set_spec(None if problem_like.spec is None else problem_like.spec.packed)
        yield ctx


_PACKED: dict = {}


def _scene_packed(scene):
    """scene.packed(), once per scene object: this repo's Scene caches its
    packing, the reference's rebuilds it on every call (geometry.py:97-98),
    which the device context would then have to re-hash to see it unchanged."""
    hit = _PACKED.get(id(scene))
    if hit is None or hit[0] is not scene:
        if len(_PACKED) > 1024:
            _PACKED.clear()
        hit = _PACKED[id(scene)] = (scene, scene.packed())
    return hit[1]


@contextmanager
def _bound_many(problem_like, devices):
    """One bound, prepared context per entry of ``devices`` (a repeated
    device gets a further independent context), every lock held."""
    from contextlib import ExitStack
    seen: dict = {}
    with ExitStack() as stack:
        ctxs = []
        for d in devices:
            slot = seen.get(d, 0)
            seen[d] = slot + 1
            c = kernels.context(problem_like.model, d, slot)
            stack.enter_context(c.lock)
            c.set_scene(_scene_packed(problem_like.scene))
            c.set_spec(None if problem_like.spec is None else problem_like.spec.packed)
            c.prepare(problem_like.params.width)
            ctxs.append(c)
        yield ctxs


def prepare(problem: PlanProblem, options: DeviceOptions = DeviceOptions()):
    """Build / load the NVRTC module for this problem's robot, constraint kind
    and width (done implicitly by plan(); call it to keep compile time out of a
    measurement, like the reference keeps file loading out of wall_ms)."""
    with _bound(problem, options) as ctx:
        ctx.prepare(problem.params.width)
    return ctx


class BatchResult(Sequence):
    """Columnar results of one batched launch (plan_many / plan_batch).

    The arrays are the decoded device output: ``codes`` (B,) int (0 Solved,
    1 TimedOut, 2 IterLimit, 3 CapacityExceeded, 5 Stopped, -1 setup error),
    ``setup_codes``, ``path_len``, ``nodes`` (B, 2), ``device_ms``, ``stats``
    (B, ST_COUNT), and every solved path packed back to back: query i's nodes
    are ``rows[offsets[i]:offsets[i + 1]]`` (FP32 tree nodes as FP64; path(i)
    puts the exact endpoints back) and its edge sources start at
    ``sources[offsets[i]]``.  Indexing gives the reference's PlanResult, built
    on first access (a 1024-query batch costs ~5 ms of Python object
    construction when every result is materialised, several times the launch
    itself)."""

    def __init__(self, a, offsets, rows, sources, starts, goals, wall_ms, single):
        # a / offsets / rows / sources are views of a result arena this object
        # holds (planner._arena): the arena is reused only once it is dropped
        self.codes = a["status"]
        self.setup_codes = a["setup_code"]
        self.path_len = np.where(self.codes == 0, a["path_len"], 0)
        self.offsets = offsets
        self.nodes = np.stack([a["ns"], a["ng"]], axis=1)
        self.device_ms = a["device_ms"]
        self.stats = a["stats"]
        self.rows, self.sources = rows, sources
        self.starts, self.goals = starts, goals
        self.wall_ms = wall_ms
        self._single = single
        self._cache: dict = {}

    def __len__(self):
        return self.codes.shape[0]

    @property
    def solved(self) -> np.ndarray:
        return self.codes == 0

    @property
    def status(self) -> list:
        return [_status_name(int(c)) for c in self.codes]

    def path(self, i: int) -> np.ndarray:
        """(L, n) path of query i; the roots are the exact FP64 endpoints."""
        o, L = int(self.offsets[i]), int(self.path_len[i])
        out = np.array(self.rows[o:o + L])
        if L:
            out[0], out[-1] = self.starts[i], self.goals[i]
        return out

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        i = range(len(self))[i]
        r = self._cache.get(i)
        if r is None:
            r = self._cache[i] = self._build(i)
        return r

    def _build(self, i):
        s = self.stats[i].tolist()
        stats = PlanStats(s[0], s[1], s[2], s[3], s[4], s[5], s[6], self.wall_ms, int(self.nodes[i, 0]),
                          int(self.nodes[i, 1]), float(self.device_ms[i]), s[8], s[9], s[10], s[11])
        code = int(self.codes[i])
        if code == 0:
            o, L = int(self.offsets[i]), int(self.path_len[i])
            return _solved(tuple(self.path(i)), tuple(map(_SRC.__getitem__, self.sources[o:o + L - 1].tolist())),
                           stats)
        if code == -1:
            if self._single:
                raise PlanSetupError(_SETUP.get(int(self.setup_codes[i]), "invalid start/goal"))
            return PlanResult("Error:PlanSetupError", None, None, stats)
        return PlanResult(_status_name(code), None, None, stats)


def _status_name(code: int) -> str:
    return "Error:PlanSetupError" if code == -1 else _STATUS.get(code, "IterLimit")


def plan_many(model, scene, spec, starts, goals, seed_offsets, params: PlanParams = PlanParams(),
              options: DeviceOptions = DeviceOptions(), devices=None) -> BatchResult:
    """Plan B independent queries of one (model, scene, spec, params) in one
    persistent launch (per device): starts / goals (B, n), seed_offsets (B,).
    The columnar form of plan_batch -- no per-query Python objects on the way
    in or out.  ``devices`` (e.g. ``range(8)``) shards the batch into
    contiguous slices, one persistent launch per device, all launched before
    any is awaited (cprrtc_plan_multi; no collective).  A device may repeat
    (independent contexts on one GPU)."""
    like = _Like(model, scene, spec, params)
    starts = np.ascontiguousarray(starts, dtype=np.float64)
    goals = np.ascontiguousarray(goals, dtype=np.float64)
    seeds = np.ascontiguousarray(seed_offsets, dtype=np.int64)
    B = starts.shape[0]
    n = model.n
    if starts.shape != (B, n) or goals.shape != (B, n) or seeds.shape != (B,):
        raise ValueError(f"starts / goals must be (B, {n}) and seed_offsets (B,)")
    if B == 0:
        raise ValueError("empty batch")
    if (seeds < 0).any():
        raise ValueError("seed_offset must be >= 0")
    prm = _params_struct(params, options)
    pc = int(prm.path_capacity)
    arena = _arena(B, pc, n)
    res, offsets, paths, srcs = arena.res, arena.offsets, arena.paths, arena.srcs
    devs = tuple(int(d) for d in devices) if devices is not None else ()
    if len(devs) > 1:
        with _bound_many(like, devs) as ctxs:
            handles = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
            t0 = time.perf_counter()
            _lib.check(ctxs[0].L.cprrtc_plan_multi(handles, len(ctxs), C.byref(prm), B, _lib.ptr(starts),
                                                   _lib.ptr(goals), _lib.ptr(seeds, _lib._lp), res,
                                                   _lib.ptr(paths), _lib.ptr(srcs, _lib._ip)), "plan_multi")
            wall = (time.perf_counter() - t0) * 1e3
        # the per-query (B, path_capacity, n) layout, packed like cprrtc_plan_flat's
        a = np.frombuffer(res, dtype=_RESULT_DT)
        L = np.where(a["status"] == 0, a["path_len"], 0)
        offsets[0] = 0
        np.cumsum(L, out=offsets[1:])
        pv, sv = paths.reshape(B, pc, n), srcs.reshape(B, pc)
        rows = np.concatenate([pv[i, :L[i]] for i in range(B)]) if L.any() else np.empty((0, n))
        srcv = np.zeros(int(offsets[B]), np.int32)
        for i in np.nonzero(L > 1)[0]:
            srcv[offsets[i]:offsets[i] + L[i] - 1] = sv[i, :L[i] - 1]
        return _batch_result(arena, res, offsets.copy(), rows, srcv, starts, goals, wall, B, pc)
    else:
        opt = options if not devs else replace(options, device=devs[0])
        with _bound(like, opt) as ctx:
            ctx.prepare(params.width)
            t0 = time.perf_counter()
            _lib.check(ctx.L.cprrtc_plan_flat(ctx.h, C.byref(prm), B, _lib.ptr(starts), _lib.ptr(goals),
                                              _lib.ptr(seeds, _lib._lp), res, _lib.ptr(offsets, _lib._lp),
                                              _lib.ptr(paths), _lib.ptr(srcs, _lib._ip), C.c_int64(B * pc)),
                       "plan")
            wall = (time.perf_counter() - t0) * 1e3
    tot = int(offsets[B])
    # no copies: the result keeps views of the arena the device results were
    # written to, and owns it until dropped
    return _batch_result(arena, res, offsets, paths[:tot], srcs[:tot], starts, goals, wall, B, pc)


def _batch_result(arena, res, offsets, rows, sources, starts, goals, wall, B, pc):
    a = np.frombuffer(res, dtype=_RESULT_DT)
    if (a["status"] == 4).any():
        raise RuntimeError(f"solution path longer than path_capacity={pc}")
    out = BatchResult(a, offsets, rows, sources, starts, goals, wall, single=(B == 1))
    out._arena = arena
    arena.owner = weakref.ref(out)
    return out


class PlanStream:
    """A stream of batches on one device (BASELINE configs[4] served
    continuously): ``submit`` launches a batch and returns at once, ``result``
    collects it as a BatchResult.  ``depth`` contexts take turns, so up to
    ``depth`` batches are in flight and a batch's slowest queries overlap the
    next batch's start (a persistent launch ends with its last query; its
    finished teams free their SMs for the next launch).  Results come back in
    submission order; each is exactly the batch plan_many would return.
    ``close()`` (or leaving a ``with`` block, or garbage collection) drains
    the batches still in flight and hands the stream's context slots to the
    next stream, so streams created one after another reuse their device
    contexts instead of accumulating them."""

    _instances = 0
    _free_bases: list = []
    _slot_lock = threading.Lock()

    def __init__(self, model, scene, spec, params: PlanParams = PlanParams(),
                 options: DeviceOptions = DeviceOptions(), depth: int = 2):
        if not 1 <= depth <= 8:
            raise ValueError("depth must be in 1..8")
        self._like = _Like(model, scene, spec, params)
        self._prm = _make_params(params, options)
        self._auto_teams = options.teams == 0
        self._pc = int(self._prm.path_capacity)
        with PlanStream._slot_lock:     # private contexts for every live stream
            if PlanStream._free_bases:
                base = PlanStream._free_bases.pop()
            else:
                PlanStream._instances += 1
                base = 1000 + 8 * PlanStream._instances
        self._ctxs = [kernels.context(model, options.device, slot=base + k) for k in range(depth)]
        for c in self._ctxs:
            with c.lock:
                c.set_scene(_scene_packed(scene))
                c.set_spec(None if spec is None else spec.packed)
                c.prepare(params.width)
        self._n = model.n
        self._next = 0
        self._inflight: dict = {}   # ticket -> (ctx, B, starts, goals, arena, t0): submitted, not collected
        self._ready: dict = {}      # ticket -> BatchResult: collected, not yet handed out
        self._finalizer = weakref.finalize(self, PlanStream._release, base, self._inflight)
        self._finalizer.atexit = False   # no device calls during interpreter shutdown

    @staticmethod
    def _release(base, inflight):
        # drain: a context holds one batch in flight and refuses the next
        # submit until it is collected (cprrtc_plan_submit)
        for ctx, B, _s, _g, arena, _t0 in list(inflight.values()):
            with ctx.lock:
                ctx.L.cprrtc_plan_wait(ctx.h, B, arena.res, _lib.ptr(arena.offsets, _lib._lp), _lib.ptr(arena.paths),
                                       _lib.ptr(arena.srcs, _lib._ip), C.c_int64(arena.srcs.shape[0]))
            arena.owner = None
        inflight.clear()
        with PlanStream._slot_lock:
            PlanStream._free_bases.append(base)

    def close(self) -> None:
        """Drain the batches still in flight and release the context slots
        (results not collected yet are dropped)."""
        self._ready.clear()
        self._finalizer()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def submit(self, starts, goals, seed_offsets) -> int:
        """Launch one batch; returns its ticket.  Blocks only when the context
        whose turn it is still holds the batch submitted ``depth`` tickets
        earlier (that one is collected first and kept for ``result``)."""
        starts = np.ascontiguousarray(starts, dtype=np.float64)
        goals = np.ascontiguousarray(goals, dtype=np.float64)
        seeds = np.ascontiguousarray(seed_offsets, dtype=np.int64)
        B = starts.shape[0]
        if B == 0 or starts.shape != (B, self._n) or goals.shape != (B, self._n) or seeds.shape != (B,):
            raise ValueError(f"starts / goals must be (B, {self._n}) and seed_offsets (B,), B >= 1")
        if (seeds < 0).any():
            raise ValueError("seed_offset must be >= 0")
        if not self._finalizer.alive:
            raise RuntimeError("PlanStream is closed")
        t = self._next
        prev = t - len(self._ctxs)
        if prev in self._inflight:
            self._ready[prev] = self._collect(prev)
        ctx = self._ctxs[t % len(self._ctxs)]
        if self._auto_teams:
            # two launches share the GPU: ~0.7 teams per query each (r2 sweep,
            # tools/batch_teams.py, 1024-query batches: 444 / 592 / 740 / 1036 /
            # 1184 / 2368 teams -> 1.10 / 1.20 / 1.29 / 1.19 / 1.02 / 0.99 M
            # queries/s end to end)
            self._prm.teams = max(64, (7 * B // 10) & ~1)
        arena = _arena(B, self._pc, self._n)
        arena.owner = lambda: ctx   # reserved until its BatchResult takes it over
        t0 = time.perf_counter()
        with ctx.lock:
            rc = ctx.L.cprrtc_plan_submit(ctx.h, C.byref(self._prm), B, _lib.ptr(starts), _lib.ptr(goals),
                                          _lib.ptr(seeds, _lib._lp))
        if rc:
            arena.owner = None
            _lib.check(rc, "plan_submit")
        self._inflight[t] = (ctx, B, starts, goals, arena, t0)
        self._next += 1
        return t

    def _collect(self, ticket):
        ctx, B, starts, goals, arena, t0 = self._inflight.pop(ticket)
        with ctx.lock:
            _lib.check(ctx.L.cprrtc_plan_wait(ctx.h, B, arena.res, _lib.ptr(arena.offsets, _lib._lp),
                                              _lib.ptr(arena.paths), _lib.ptr(arena.srcs, _lib._ip),
                                              C.c_int64(B * self._pc)), "plan_wait")
        wall = (time.perf_counter() - t0) * 1e3
        tot = int(arena.offsets[B])
        return _batch_result(arena, arena.res, arena.offsets, arena.paths[:tot], arena.srcs[:tot], starts, goals,
                             wall, B, self._pc)

    def result(self, ticket: int) -> "BatchResult":
        """The BatchResult of ``ticket`` (waits for it if still in flight)."""
        if ticket in self._ready:
            return self._ready.pop(ticket)
        if ticket in self._inflight:
            return self._collect(ticket)
        raise KeyError(f"unknown or already collected ticket {ticket}")


class _Like:
    """The (model, scene, spec, params) a context is bound to."""

    __slots__ = ("model", "scene", "spec", "params")

    def __init__(self, model, scene, spec, params):
        self.model, self.scene, self.spec, self.params = model, scene, spec, params


def plan_batch(problems, options: DeviceOptions = DeviceOptions(), return_dense: bool = False,
               devices=None):
    """Plan many independent queries in one persistent launch (plan_many on
    the problems' starts, goals and seeds).

    All problems must share model, scene, spec and params (apart from
    start, goal and params.seed_offset).  Returns a BatchResult (a sequence
    of PlanResult, built lazily); a bad start/goal raises PlanSetupError for
    that problem only if it is the sole problem, else its result carries
    status 'Error:PlanSetupError'.  ``devices``: as for plan_many.
    """
    problems = list(problems)
    if not problems:
        return []
    p0 = problems[0]
    if len(problems) > 1:
        key = _params_getter()
        base = key(p0.params)
        for p in problems[1:]:
            if (p.model is not p0.model or p.scene is not p0.scene or p.spec is not p0.spec
                    or (p.params is not p0.params and key(p.params) != base)):
                raise ValueError("plan_batch problems must share model, scene, spec and params")
    out = plan_many(p0.model, p0.scene, p0.spec, np.stack([p.start for p in problems]),
                    np.stack([p.goal for p in problems]), [int(p.params.seed_offset) for p in problems],
                    p0.params, options, devices)
    if return_dense:
        out = list(out)
        prm = _params_struct(p0.params, options)
        with _bound(p0, options) as ctx:
            for i, r in enumerate(out):
                if r.solved and len(r.path) > 1:
                    src = np.array([_SRC.index(x) for x in r.edge_sources], np.int32)
                    dense, ok = _derive(ctx, prm, np.stack(r.path), src)
                    out[i] = replace(r, dense=dense)
    return out


_PARAMS_GETTER = None


def _params_getter():
    """PlanParams fields except seed_offset, as one C-level attrgetter
    (plan_batch's consistency check)."""
    global _PARAMS_GETTER
    if _PARAMS_GETTER is None:
        from dataclasses import fields
        from operator import attrgetter
        _PARAMS_GETTER = attrgetter(*(f.name for f in fields(PlanParams) if f.name != "seed_offset"))
    return _PARAMS_GETTER


_RESULT_DT = np.dtype({"names": ["status", "setup_code", "path_len", "ns", "ng", "device_ms", "stats"],
                       "formats": [np.int32, np.int32, np.int32, np.int32, np.int32, np.float64,
                                   (np.uint64, _lib.ST_COUNT)],
                       "offsets": [_lib.Result.status.offset, _lib.Result.setup_code.offset,
                                   _lib.Result.path_len.offset, _lib.Result.nodes_start.offset,
                                   _lib.Result.nodes_goal.offset, _lib.Result.device_ms.offset,
                                   _lib.Result.stats.offset],
                       "itemsize": C.sizeof(_lib.Result)})


def _solved(path, sources, stats) -> "PlanResult":
    """PlanResult("Solved", path, sources, stats) without the frozen
    dataclass's per-field __setattr__ round trips (the batch decoding loop
    builds one per query)."""
    r = object.__new__(PlanResult)
    r.__dict__.update(status="Solved", path=path, edge_sources=sources, stats=stats, dense=None)
    return r


_SRC_CACHE: dict = {}


def _sources(srcs_i, L) -> tuple:
    """Edge-source names of a path (the codes' bytes key a small cache: a
    path's sources are start edges, a junction, goal edges)."""
    key = srcs_i[:L - 1].tobytes()
    t = _SRC_CACHE.get(key)
    if t is None:
        if len(_SRC_CACHE) > 4096:
            _SRC_CACHE.clear()
        t = _SRC_CACHE[key] = tuple(map(_SRC.__getitem__, srcs_i[:L - 1].tolist()))
    return t


def _result_one(r, p, paths_i, srcs_i, wall, pc) -> "PlanResult":
    """The single-query latency path's decoding (one ctypes result; the C
    call wrote the exact FP64 endpoints into the path's first and last rows)."""
    s = r.stats[:]
    stats = PlanStats(s[0], s[1], s[2], s[3], s[4], s[5], s[6], wall, r.nodes_start, r.nodes_goal,
                      r.device_ms, s[8], s[9], s[10], s[11])
    code = r.status
    if code == 0:
        L = r.path_len
        rows = paths_i[:L].copy()                # one array; the path's nodes are its rows
        return _solved(tuple(rows), _sources(srcs_i, L), stats)
    if code == -1:
        raise PlanSetupError(_SETUP.get(r.setup_code, "invalid start/goal"))
    if code == 4:
        raise RuntimeError(f"solution path longer than path_capacity={pc}")
    return PlanResult(_STATUS.get(code, "IterLimit"), None, None, stats)


def _result(r, p, paths_i, srcs_i, wall, B, pc) -> PlanResult:
    """PlanResult of one cprrtc_result (paths_i (pc, n), srcs_i (pc,))."""
    st = r.stats
    stats = PlanStats(iterations=int(st[0]), extensions_attempted=int(st[1]),
                      extensions_added=int(st[2]), projection_failures=int(st[3]),
                      collision_rejections=int(st[4]), cc_performed=int(st[5]),
                      cc_possible=int(st[6]), wall_ms=wall, nodes_start=int(r.nodes_start),
                      nodes_goal=int(r.nodes_goal), device_ms=float(r.device_ms),
                      stage1_evals=int(st[8]), cc_fk_evals=int(st[9]), nn_nodes=int(st[10]),
                      proj_iters=int(st[11]))
    if r.status == -1:
        if B == 1:
            raise PlanSetupError(_SETUP.get(r.setup_code, "invalid start/goal"))
        return PlanResult("Error:PlanSetupError", None, None, stats)
    if r.status == 4:
        raise RuntimeError(f"solution path longer than path_capacity={pc}")
    if r.status != 0:
        return PlanResult(_STATUS.get(r.status, "IterLimit"), None, None, stats)
    L = int(r.path_len)
    path = list(paths_i[:L].copy())
    path[0] = p.start.copy()                 # roots are the exact FP64 endpoints
    path[-1] = p.goal.copy()
    sources = tuple(_SRC[int(k)] for k in srcs_i[:L - 1])
    return PlanResult("Solved", tuple(path), sources, stats)


class _Session:
    """One thread's bound single-query call for one (model, scene, spec,
    options): context, the scene / constraint packings, the parameter block of
    the last PlanParams seen (every query usually carries its own PlanParams,
    differing only in seed_offset, which travels separately) and reusable host
    buffers with their ctypes pointers, so the latency path builds no arrays
    and looks nothing up twice per call."""

    __slots__ = ("objs", "ctx", "params", "pkey", "prm", "pc", "width", "pscene", "pspec", "s", "g", "seed",
                 "res", "paths", "srcs", "args", "fast")

    def __init__(self, problem, options):
        self.objs = (problem.model, problem.scene, problem.spec, options)
        self.ctx = kernels.context(problem.model, options.device)
        self.pscene = _scene_packed(problem.scene)
        self.pspec = None if problem.spec is None else problem.spec.packed
        self.params = self.pkey = None
        self.pc = -1
        n = self.ctx.n
        self.s = np.empty((1, n))
        self.g = np.empty((1, n))
        self.seed = np.zeros(1, np.int64)
        self.res = (_lib.Result * 1)()

    def use(self, params, options):
        """Bind params (re-deriving the parameter block only when a field
        other than seed_offset changed)."""
        if params is self.params:
            return
        key = _params_getter()(params)
        if key != self.pkey:
            self.prm = _make_params(params, options)
            self.width = params.width
            pc = int(self.prm.path_capacity)
            if pc != self.pc:
                self.pc = pc
                self.paths = np.empty((1, pc, self.ctx.n))
                self.srcs = np.empty((1, pc), np.int32)
            self.args = (self.ctx.h, C.byref(self.prm), 1, _lib.ptr(self.s), _lib.ptr(self.g),
                         _lib.ptr(self.seed, _lib._lp), self.res, _lib.ptr(self.paths), _lib.ptr(self.srcs, _lib._ip))
            # the _cprrtc_fast arguments around (start, goal, seed): the same buffers by address
            self.fast = (self.ctx.h.value, C.addressof(self.prm), C.addressof(self.res), self.paths.ctypes.data,
                         self.srcs.ctypes.data, self.ctx.n)
            self.pkey = key
        self.params = params


_TLS = threading.local()


def _session(problem, options) -> _Session:
    cache = getattr(_TLS, "sessions", None)
    if cache is None:
        cache = _TLS.sessions = {}
    key = (id(problem.model), id(problem.scene), id(problem.spec), id(options))
    s = cache.get(key)
    if s is None or s.objs[0] is not problem.model or s.objs[1] is not problem.scene \
            or s.objs[2] is not problem.spec or s.objs[3] is not options:
        if len(cache) > 256:
            cache.clear()
        s = cache[key] = _Session(problem, options)
    s.use(problem.params, options)
    return s


_FAST_UNSET = object()
_FAST = _FAST_UNSET


def _fast():
    """The CPython fast path of the single-query call (csrc/pyfast.c), or
    None (not built, or CPRRTC_NO_FAST=1): then plan() goes through ctypes."""
    global _FAST
    if _FAST is _FAST_UNSET:
        f = None
        if os.environ.get("CPRRTC_NO_FAST", "0") in ("", "0"):
            try:
                from . import _cprrtc_fast as f
                f.setup(C.cast(_lib.load().cprrtc_plan, C.c_void_p).value, _SRC)
            except ImportError:
                f = None
        _FAST = f
    return _FAST


def _result_fast(out, pc) -> "PlanResult":
    """PlanResult of a _cprrtc_fast.plan_one tuple (0, status, setup_code,
    stats in PlanStats order, path rows, sources)."""
    code = out[1]
    stats = PlanStats(*out[3])
    if code == 0:
        return _solved(out[4], out[5], stats)
    if code == -1:
        raise PlanSetupError(_SETUP.get(out[2], "invalid start/goal"))
    if code == 4:
        raise RuntimeError(f"solution path longer than path_capacity={pc}")
    return PlanResult(_STATUS.get(code, "IterLimit"), None, None, stats)


def _plan_one(problem: PlanProblem, options: DeviceOptions, return_dense: bool) -> PlanResult:
    ss = _session(problem, options)
    seed = problem.params.seed_offset
    if seed < 0:
        raise ValueError("seed_offset must be >= 0")
    ctx = ss.ctx
    fast = _FAST if _FAST is not _FAST_UNSET else _fast()
    with ctx.lock:   # bind + launch under one lock (planner._bound)
        ctx.set_scene(ss.pscene)
        ctx.set_spec(ss.pspec)
        ctx.prepare(ss.width)
        out = None
        if fast is not None:
            h, prm, res, paths, srcs, n = ss.fast
            out = fast.plan_one(h, prm, problem.start, problem.goal, seed, res, paths, srcs, n)
        if out is not None:
            if out[0]:
                _lib.check(out[0], "plan")
            res = _result_fast(out, ss.pc)
        else:   # ctypes (no fast module, or inputs it does not take: not float64 C-contiguous)
            ss.s[0] = problem.start
            ss.g[0] = problem.goal
            ss.seed[0] = seed
            t0 = time.perf_counter()
            rc = ctx.L.cprrtc_plan(*ss.args)
            wall = (time.perf_counter() - t0) * 1e3
            if rc:
                _lib.check(rc, "plan")
            res = _result_one(ss.res[0], problem, ss.paths[0], ss.srcs[0], wall, ss.pc)
        if return_dense and res.solved:
            L = len(res.path)
            dense, ok = _derive(ctx, ss.prm, ss.paths[0, :L], ss.srcs[0, :L - 1])
            res = replace(res, dense=dense)
    return res


class _Arena:
    """Host result buffers of one batch launch: the result structs, path
    offsets (B+1), and the packed path rows / sources sized for the worst case
    B * path_capacity (virtual memory: only the rows a batch writes are ever
    touched).  The BatchResult built on it keeps views and owns it; a later
    call reuses it only after that result is gone (no copy-out, no fresh
    page faults per call).  "Gone" includes every view of the buffers a
    caller kept (``r.rows``, ``r.codes``, ... outliving ``r``): each view holds
    a reference to its buffer, so the buffers' reference counts must be back
    at their resting values before the arena is handed out again."""

    __slots__ = ("res", "offsets", "paths", "srcs", "owner", "_rest")

    def __init__(self, B, pc, n):
        self.res = (_lib.Result * B)()
        self.offsets = np.zeros(B + 1, np.int64)
        self.paths = np.empty((B * pc, n))
        self.srcs = np.empty(B * pc, np.int32)
        self.owner = None
        self._rest = self._refs()

    def _refs(self):
        return (sys.getrefcount(self.res), sys.getrefcount(self.offsets), sys.getrefcount(self.paths),
                sys.getrefcount(self.srcs))

    def free(self) -> bool:
        """No owner alive and no outstanding view of any buffer."""
        return (self.owner is None or self.owner() is None) and self._refs() == self._rest


def _arena(B, pc, n) -> _Arena:
    pools = getattr(_TLS, "arenas", None)
    if pools is None:
        pools = _TLS.arenas = {}
    pool = pools.setdefault((B, pc, n), [])
    for a in pool:
        if a.free():
            a.owner = None
            return a
    a = _Arena(B, pc, n)
    if len(pool) < 4:
        pool.append(a)
    return a


def plan(problem: PlanProblem, options: DeviceOptions = DeviceOptions(),
         return_dense: bool = False) -> PlanResult:
    """reference plan() (planner.py:430-485) on the device."""
    # start == goal (np.array_equal semantics: -0.0 == 0.0, NaN != NaN) through
    # Python float lists: ~10x cheaper than array_equal on the latency path
    if problem.start.tolist() == problem.goal.tolist():
        # endpoint checks first, exactly like the reference (planner.py:435-440)
        t0 = time.perf_counter()
        code = kernels.check_config_batch(problem.model, problem.scene, problem.spec,
                                          problem.start[None], _tau(problem), options.device)[0]
        if code:
            raise PlanSetupError(_SETUP[int(code)])
        stats = PlanStats(wall_ms=(time.perf_counter() - t0) * 1e3, nodes_start=1, nodes_goal=1)
        return PlanResult("Solved", (problem.start.copy(),), (), stats)
    return _plan_one(problem, options, return_dense)


RACE_SEED_STRIDE = 1_000_000_007   # Halton offset between racers (distinct sample streams)


def plan_race(problem: PlanProblem, devices=(0, 1), options: DeviceOptions = DeviceOptions()):
    """One query raced on several GPUs (cprrtc_plan_race): racer k plans on
    ``devices[k]`` with seed_offset + k * RACE_SEED_STRIDE; the first to solve
    stores a first-solution flag into every racer's flag word over NVLink
    (peer stores) and the others stop.  Returns (PlanResult of the winner, or
    of racer 0 if none solved, winner index or -1, per-racer PlanResults).
    A device may appear more than once (independent contexts on one GPU)."""
    devices = tuple(int(d) for d in devices)
    if not 1 <= len(devices) <= _lib.MAX_RACE:
        raise ValueError(f"1..{_lib.MAX_RACE} racers")
    if np.array_equal(problem.start, problem.goal):
        r = plan(problem, replace(options, device=devices[0]))
        return r, 0, [r]
    prm = _params_struct(problem.params, options)
    base = int(problem.params.seed_offset)
    if base < 0:
        raise ValueError("seed_offset must be >= 0")
    R = len(devices)
    pc = int(prm.path_capacity)
    n = problem.model.n
    seeds = np.array([base + k * RACE_SEED_STRIDE for k in range(R)], np.int64)
    start = np.ascontiguousarray(problem.start, dtype=np.float64)
    goal = np.ascontiguousarray(problem.goal, dtype=np.float64)
    res = (_lib.Result * R)()
    paths = np.empty((R, pc, n))
    srcs = np.empty((R, pc), np.int32)
    win = C.c_int32(-1)
    with _bound_many(problem, devices) as ctxs:
        handles = (C.c_void_p * R)(*[c.h.value for c in ctxs])
        t0 = time.perf_counter()
        _lib.check(ctxs[0].L.cprrtc_plan_race(handles, R, C.byref(prm), _lib.ptr(start), _lib.ptr(goal),
                                              _lib.ptr(seeds, _lib._lp), res, _lib.ptr(paths),
                                              _lib.ptr(srcs, _lib._ip), C.byref(win)), "plan_race")
        wall = (time.perf_counter() - t0) * 1e3
    per = [_result(res[k], problem, paths[k], srcs[k], wall, 1, pc) for k in range(R)]
    w = int(win.value)
    return per[w if w >= 0 else 0], w, per


def _tau(problem) -> float:
    pp = problem.params.projection
    if pp.tau_task is not None:
        return float(pp.tau_task)
    return math.inf if problem.spec is None else float(problem.spec.tau_task)


def _derive(ctx, prm, nodes, sources):
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    sources = np.ascontiguousarray(sources, dtype=np.int32)
    E = nodes.shape[0] - 1
    W = int(prm.width)
    dense = np.empty((max(E, 0), W, ctx.n))
    ok = np.empty(max(E, 0), np.int32)
    if E > 0:
        with ctx.lock:
            _lib.check(ctx.L.cprrtc_derive_edges(ctx.h, C.byref(prm), nodes.shape[0],
                                                 _lib.ptr(nodes), _lib.ptr(sources, _lib._ip),
                                                 _lib.ptr(dense), _lib.ptr(ok, _lib._ip)),
                       "derive_edges")
    return dense, ok.astype(bool)


def derive_edge(a, b, ctx: PlanContext, stats: PlanStats | None = None):
    """The re-derivable motion a -> b (planner.py:223-245) or None; device."""
    spec = None if ctx.spec is not None and math.isinf(ctx.spec.tau_task) else ctx.spec
    prob = PlanProblem(ctx.model, ctx.scene, spec, a, b, ctx.params)
    prm = _params_struct(ctx.params, ctx.options)
    with _bound(prob, ctx.options) as dctx:
        dense, ok = _derive(dctx, prm, np.stack([prob.start, prob.goal]), np.zeros(1, np.int32))
    return MotionSegment(dense[0]) if ok[0] else None


def derive_path(result: PlanResult, problem: PlanProblem,
                options: DeviceOptions = DeviceOptions()):
    """Every edge of a solved path re-derived on the device exactly as the
    planner certified it: (dense (E, W, n), ok (E,))."""
    prm = _params_struct(problem.params, options)
    src = np.array([_SRC.index(s) for s in result.edge_sources], dtype=np.int32)
    with _bound(problem, options) as ctx:
        return _derive(ctx, prm, np.stack(result.path), src)


def revalidate_path(result: PlanResult, problem: PlanProblem,
                    options: DeviceOptions = DeviceOptions()) -> bool:
    """Re-derive and re-check every edge of a solved path on the device
    (planner.py:508-523).  For a path returned by plan() this reproduces the
    certified motions exactly (same FP32 inputs, same kernels)."""
    if not result.solved:
        return False
    if len(result.path) < 2:
        return True
    return bool(derive_path(result, problem, options)[1].all())


def dense_path(result: PlanResult, problem: PlanProblem,
               options: DeviceOptions = DeviceOptions()) -> np.ndarray:
    """Dense waypoints (E*(W-1)+1, n) of a solved path, re-derived on the
    device; consecutive edges share their junction waypoint."""
    if len(result.path) < 2:
        return np.stack(result.path)
    dense, ok = derive_path(result, problem, options)
    if not ok.all():
        raise RuntimeError("a path edge failed device re-derivation")
    return np.concatenate([dense[0]] + [d[1:] for d in dense[1:]])


def extract_path(tree_s: Tree, tree_g: Tree, meet_s: int, meet_g: int):
    """Host path assembly on Tree objects (planner.py:488-505 contract)."""
    pa = [tree_s.node(i) for i in tree_s.chain(meet_s)]
    pb = [tree_g.node(i) for i in reversed(tree_g.chain(meet_g))]
    sources = ["start"] * (len(pa) - 1)
    dup = np.array_equal(pa[-1], pb[0])
    if dup:
        pb = pb[1:]
    if pb:
        sources.append("goal" if dup else "junction")
        sources += ["goal"] * (len(pb) - 1)
    return tuple(pa + pb), tuple(sources)


_REASON = {-1: "degenerate", -2: "projection", -3: "collision", -4: "capacity"}


def _step(op: int, tree: Tree, q, ctx: PlanContext):
    spec = None if ctx.spec is not None and math.isinf(ctx.spec.tau_task) else ctx.spec
    n = tree.nodes.shape[1]
    q = np.ascontiguousarray(np.asarray(q, dtype=float).reshape(n))
    prob = PlanProblem(ctx.model, ctx.scene, spec, tree.node(0), tree.node(0), ctx.params)
    prm = _params_struct(ctx.params, ctx.options)
    nodes = np.ascontiguousarray(tree.nodes, dtype=np.float64)
    parents = np.ascontiguousarray(tree.parents, dtype=np.int32)
    res = np.zeros(3, np.int32)
    cap_new = int(ctx.params.max_connect_segments) + 2
    new_nodes = np.empty((cap_new, n))
    new_par = np.empty(cap_new, np.int32)
    st = np.zeros(_lib.ST_COUNT, np.uint64)
    with _bound(prob, ctx.options) as dctx:
        dctx.prepare(ctx.params.width)
        _lib.check(dctx.L.cprrtc_step(dctx.h, C.byref(prm), op, len(tree), _lib.ptr(nodes),
                                      _lib.ptr(parents, _lib._ip), _lib.ptr(q), _lib.ptr(res, _lib._ip),
                                      _lib.ptr(new_nodes), _lib.ptr(new_par, _lib._ip), cap_new,
                                      st.ctypes.data_as(C.POINTER(C.c_uint64))), "step")
    added = int(res[2]) - len(tree)
    for i in range(added):
        tree.add(new_nodes[i], int(new_par[i]))
    s = ctx.stats
    s.extensions_attempted += int(st[1])
    s.extensions_added += int(st[2])
    s.projection_failures += int(st[3])
    s.collision_rejections += int(st[4])
    s.cc_performed += int(st[5])
    s.cc_possible += int(st[6])
    return int(res[0]), int(res[1]), added


def extend(tree: Tree, q_rand, ctx: PlanContext) -> ExtendOutcome:
    """One projected extension toward a sample (planner.py:317-325), on the
    device; the tree gains the node on success."""
    r, _, _ = _step(0, tree, q_rand, ctx)
    if r >= 0:
        return ExtendOutcome("Added", node=r)
    return ExtendOutcome("Rejected", reason=_REASON[r])


def connect(tree: Tree, q_target, ctx: PlanContext) -> ConnectOutcome:
    """Greedy connect toward a target (planner.py:361-409), on the device."""
    r, segs, added = _step(1, tree, q_target, ctx)
    if r >= 0:
        return ConnectOutcome("Reached", node=r, segments=segs)
    if segs > 0:
        return ConnectOutcome("Advanced", node=len(tree) - 1, segments=segs)
    return ConnectOutcome("Trapped", node=None, segments=0)


def _check_endpoint_message(code: int) -> str:
    return _SETUP[code]


def task_error_norm(problem: PlanProblem, q) -> float:
    e = task_error(problem.spec if problem.spec is not None else unconstrained(),
                   forward_kinematics(problem.model, q))
    return float(np.sqrt((e * e).sum()))
