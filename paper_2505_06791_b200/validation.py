"""Motion validation with the early-termination flag (device).

Mirrors ``maniplan/validation.py``.  One team per motion, lane t = waypoint
t; lanes step through the reference's check order in lockstep and vote every
CP_CHUNK checks (the paper's shared collision flag), so the
verdict, the first colliding waypoint and the lockstep-equivalent
``primitive_checks_performed`` equal the reference's
(``maniplan/_kernels/pure.py:646-699``) up to FP32 contacts within 1e-5 m.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import kernels
from .projection import MotionSegment

__all__ = ["ValidationReport", "validate_motion", "validate_configuration"]


@dataclass(frozen=True)
class ValidationReport:
    valid: bool
    primitive_checks_performed: int
    primitive_checks_possible: int
    first_colliding_waypoint: int | None

    @property
    def checks_saved(self) -> int:
        return self.primitive_checks_possible - self.primitive_checks_performed


def _waypoints(seg) -> np.ndarray:
    if isinstance(seg, MotionSegment):
        return seg.waypoints
    wp = np.asarray(seg, dtype=float)
    if wp.ndim != 2:
        raise ValueError("expected a MotionSegment or (W, n) array")
    return wp


def validate_motion(seg, scene, model, flag_mode: str = "on",
                    execution: str = "deterministic") -> ValidationReport:
    wp = _waypoints(seg)
    if wp.shape[1] != model.n:
        raise ValueError("waypoint dimension does not match the model")
    if flag_mode not in ("on", "off"):
        raise ValueError(f"flag_mode must be 'on' or 'off', got {flag_mode!r}")
    if execution not in ("deterministic", "threaded"):
        raise ValueError(f"unknown execution {execution!r}")
    r = kernels.validate_batch(model, scene, wp[None], flag_mode == "on")
    fb = int(r["first_bad"][0])
    return ValidationReport(bool(r["valid"][0]), int(r["performed"][0]), int(r["possible"][0]),
                            None if fb < 0 else fb)


def validate_configuration(q, scene, model) -> bool:
    """Collision-free test of one configuration (FP64 on the device)."""
    q = model.check_q(q)
    code = kernels.check_config_batch(model, scene, None, q[None], float("inf"))[0]
    if code == 1:
        # the reference does not test limits here; re-run without them
        r = kernels.validate_batch(model, scene, q[None, None, :], False)
        return bool(r["valid"][0])
    return code == 0
