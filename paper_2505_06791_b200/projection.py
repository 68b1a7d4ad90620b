"""Motion segments and their projection onto the constraint manifold.

Mirrors ``maniplan/projection.py``.  ``parallel_project`` runs Alg. 1 (the
paper's parallel projection operator) on the device: one
team of lanes, lane t owning waypoint t, stage 2 a warp ballot
(``cp_project`` in csrc/device/cprrtc_device.cuh); ``sequential_project``
runs the CBiRRT-style baseline on the device; ``project_configuration`` is
an FP64 device Newton solve.  ``interpolate_segment`` and ``segment_gaps``
are host-side segment constructors, as in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import kernels

__all__ = [
    "MotionSegment", "ProjectionParams", "ProjectionOutcome", "IterationSnapshot",
    "interpolate_segment", "parallel_project", "sequential_project",
    "project_configuration", "segment_gaps", "MODE_NAMES",
]

MODE_NAMES = {"parallel": 0, "literal-gap": 1, "naive": 2}
_TAU_SM_SCALE = 1.5
_TAU_SM_FLOOR = 1e-6


@dataclass(frozen=True)
class MotionSegment:
    """(W, n) waypoints; row 0 is the fixed start."""

    waypoints: np.ndarray

    def __post_init__(self):
        wp = np.ascontiguousarray(np.asarray(self.waypoints, dtype=float))
        if wp.ndim != 2 or wp.shape[0] < 2:
            raise ValueError("waypoints must be (W, n) with W >= 2")
        object.__setattr__(self, "waypoints", wp)

    @property
    def width(self) -> int:
        return self.waypoints.shape[0]

    @property
    def dim(self) -> int:
        return self.waypoints.shape[1]

    @property
    def start(self) -> np.ndarray:
        return self.waypoints[0]

    @property
    def end(self) -> np.ndarray:
        return self.waypoints[-1]


@dataclass(frozen=True)
class ProjectionParams:
    alpha: float = 0.1
    max_iters: int = 128
    lam: float = 1e-3
    tau_task: float | None = None
    tau_sm: float | None = None

    def __post_init__(self):
        if self.alpha <= 0 or self.lam < 0 or self.max_iters < 1:
            raise ValueError("alpha > 0, lam >= 0, max_iters >= 1 required")
        for tau in (self.tau_task, self.tau_sm):
            if tau is not None and not tau > 0:
                raise ValueError("tolerances must be positive")


@dataclass(frozen=True)
class IterationSnapshot:
    iteration: int
    prog: int
    waypoints: np.ndarray


@dataclass(frozen=True)
class ProjectionOutcome:
    status: str              # Projected | Failed
    segment: MotionSegment
    iterations_used: int
    final_prog: int
    trace: tuple | None = field(default=None, compare=False)

    @property
    def ok(self) -> bool:
        return self.status == "Projected"


def interpolate_segment(a, b, width: int) -> MotionSegment:
    """Straight line with ``width`` waypoints; endpoints stored exactly."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.ndim != 1 or a.shape != b.shape:
        raise ValueError("endpoints must be 1-D and the same length")
    if width < 2:
        raise ValueError("width must be >= 2")
    frac = np.arange(width, dtype=float) / (width - 1)
    wp = a[None, :] + frac[:, None] * (b - a)[None, :]
    wp[0] = a
    wp[-1] = b
    return MotionSegment(wp)


def segment_gaps(seg: MotionSegment) -> np.ndarray:
    d = np.diff(seg.waypoints, axis=0)
    return np.sqrt((d * d).sum(axis=1))


def _taus(seg, spec, params):
    tau_task = params.tau_task if params.tau_task is not None else spec.tau_task
    if params.tau_sm is not None:
        return float(tau_task), float(params.tau_sm)
    gap = float(segment_gaps(seg).max())
    return float(tau_task), (_TAU_SM_SCALE * gap if gap > 0 else _TAU_SM_FLOOR)


def _run(seg, spec, model, params, mode, collect_trace):
    if seg.dim != model.n:
        raise ValueError("segment dimension does not match the model")
    tau_task, tau_sm = _taus(seg, spec, params)
    packed_spec = None if math.isinf(tau_task) and math.isinf(spec.tau_task) else spec.packed
    r = kernels.project_batch(model, packed_spec if packed_spec is not None else spec.packed,
                              seg.waypoints[None], tau_task, tau_sm, params.alpha, params.lam,
                              params.max_iters, mode, collect_trace)
    trace = None
    if collect_trace and r["trace"] is not None:
        tp = r["trace_prog"][0]
        k = int((tp >= 0).sum())
        trace = tuple(IterationSnapshot(i + 1, int(tp[i]), r["trace"][0, i].copy())
                      for i in range(k))
    ok = bool(r["ok"][0])
    return ProjectionOutcome("Projected" if ok else "Failed", MotionSegment(r["xi"][0]),
                             int(r["iters"][0]), int(r["prog"][0]), trace)


def parallel_project(seg: MotionSegment, spec, model, params: ProjectionParams,
                     mode: str = "parallel", collect_trace: bool = False,
                     execution: str = "deterministic") -> ProjectionOutcome:
    """Alg. 1 on the device (FP32, clamp-and-revalidate finish included).

    ``execution`` is accepted for API parity; the device team is the real
    concurrent worker team and is iteration-deterministic by construction.
    """
    if mode == "naive":
        return sequential_project(seg, spec, model, params)
    if mode not in MODE_NAMES:
        raise ValueError(f"unknown projection mode {mode!r}")
    if execution not in ("deterministic", "threaded"):
        raise ValueError(f"unknown execution {execution!r}")
    return _run(seg, spec, model, params, MODE_NAMES[mode], collect_trace)


def sequential_project(seg: MotionSegment, spec, model, params: ProjectionParams) -> ProjectionOutcome:
    return _run(seg, spec, model, params, 2, False)


def project_configuration(q, spec, model, tau_task: float | None = None, lam: float = 1e-3,
                          max_iters: int = 128):
    """FP64 device Newton projection of one configuration -> (q, ok)."""
    q = model.check_q(q)
    tau = float(tau_task if tau_task is not None else spec.tau_task)
    out, ok = kernels.project_config_batch(model, spec, q[None], tau, lam, max_iters)
    return out[0], bool(ok[0])
