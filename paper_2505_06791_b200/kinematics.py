"""Serial-chain robot model, its packed layout, and device-backed FK.

Public names mirror ``maniplan/kinematics.py`` (Joint, LinkSphere,
RobotModel, PackedRobot, FrameSet, forward_kinematics ...; YAML loading is
the reference's own).
``RobotModel.packed`` reproduces the reference packing bit-for-bit
(``kinematics.py:176-224``); the device never sees these float64 arrays
directly -- the NVRTC code generator folds them into unrolled FP32 FK code
(``csrc/codegen.cpp``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property
from math import cos, sin

import numpy as np

from .geometry import Sphere

__all__ = [
    "Joint", "LinkSphere", "RobotModel", "FrameSet", "PackedRobot",
    "forward_kinematics", "collision_spheres_world", "geometric_jacobian",
    "load_robot", "dump_robot", "clamp_to_limits", "robot_from_dict",
]

_UNIT_TOL = 1e-9


@dataclass(frozen=True)
class Joint:
    jtype: str
    axis: np.ndarray
    origin_xyz: np.ndarray
    origin_rpy: np.ndarray
    lo: float
    hi: float
    name: str = ""

    def __post_init__(self):
        for attr in ("axis", "origin_xyz", "origin_rpy"):
            object.__setattr__(self, attr, np.asarray(getattr(self, attr), dtype=float))
        if self.jtype not in ("revolute", "prismatic"):
            raise ValueError(f"unknown joint type {self.jtype!r}")
        if abs(float(np.linalg.norm(self.axis)) - 1.0) > _UNIT_TOL:
            raise ValueError("joint axis must be unit-norm")
        if not self.lo < self.hi:
            raise ValueError("joint limits must satisfy lo < hi")


@dataclass(frozen=True)
class LinkSphere:
    link: int
    center: np.ndarray
    radius: float

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=float))
        if self.radius <= 0:
            raise ValueError("sphere radius must be positive")


@dataclass(frozen=True)
class PackedRobot:
    """Reference packed layout (kinematics.py:158-173)."""

    jtypes: np.ndarray        # (n,) int32, 0 revolute / 1 prismatic
    axes: np.ndarray          # (n, 3)
    origin_r: np.ndarray      # (n, 9) row-major Rz*Ry*Rx of the origin rpy
    origin_p: np.ndarray      # (n, 3)
    lo: np.ndarray            # (n,)
    hi: np.ndarray            # (n,)
    sphere_link: np.ndarray   # (S,) int32
    sphere_local: np.ndarray  # (S, 3)
    sphere_radius: np.ndarray  # (S,)
    pairs: np.ndarray         # (P, 2) int32
    ee_link: int

    @property
    def n(self) -> int:
        return int(self.jtypes.shape[0])


def rpy_to_matrix(roll: float, pitch: float, yaw: float) -> tuple:
    """Fixed-axis roll/pitch/yaw -> row-major R = Rz(yaw) Ry(pitch) Rx(roll)."""
    cr, sr = cos(roll), sin(roll)
    cp, sp = cos(pitch), sin(pitch)
    cy, sy = cos(yaw), sin(yaw)
    row0 = (cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr)
    row1 = (sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr)
    row2 = (-sp, cp * sr, cp * cr)
    return row0 + row1 + row2


@dataclass(frozen=True)
class RobotModel:
    joints: tuple
    link_spheres: tuple = ()
    ee_link: int = -1
    self_collision_pairs: tuple = ()
    name: str = ""
    zero_pose_ee: np.ndarray | None = field(default=None, compare=False)

    def __post_init__(self):
        n = len(self.joints)
        if n == 0:
            raise ValueError("a robot needs at least one joint")
        ee = n - 1 if self.ee_link < 0 else self.ee_link
        if not 0 <= ee < n:
            raise ValueError(f"ee_link {self.ee_link} out of range for {n} joints")
        object.__setattr__(self, "ee_link", ee)
        object.__setattr__(self, "joints", tuple(self.joints))
        object.__setattr__(self, "link_spheres", tuple(self.link_spheres))
        object.__setattr__(self, "self_collision_pairs",
                           tuple(tuple(int(v) for v in p) for p in self.self_collision_pairs))
        for k, s in enumerate(self.link_spheres):
            if not 0 <= s.link < n:
                raise ValueError(f"link_spheres[{k}].link out of range")
        ns = len(self.link_spheres)
        for k, (i, j) in enumerate(self.self_collision_pairs):
            if i == j or not (0 <= i < ns and 0 <= j < ns):
                raise ValueError(f"self_collision_pairs[{k}] invalid")
        if self.zero_pose_ee is not None:
            object.__setattr__(self, "zero_pose_ee", np.asarray(self.zero_pose_ee, dtype=float))

    @property
    def n(self) -> int:
        return len(self.joints)

    @property
    def limits(self) -> np.ndarray:
        return np.array([[j.lo, j.hi] for j in self.joints])

    @cached_property
    def packed(self) -> PackedRobot:
        n, ns, npair = self.n, len(self.link_spheres), len(self.self_collision_pairs)
        c = np.ascontiguousarray
        return PackedRobot(
            jtypes=c(np.array([int(j.jtype != "revolute") for j in self.joints], dtype=np.int32)),
            axes=c(np.array([j.axis for j in self.joints], dtype=float).reshape(n, 3)),
            origin_r=c(np.array([rpy_to_matrix(*j.origin_rpy) for j in self.joints]).reshape(n, 9)),
            origin_p=c(np.array([j.origin_xyz for j in self.joints], dtype=float).reshape(n, 3)),
            lo=c(np.array([j.lo for j in self.joints], dtype=float)),
            hi=c(np.array([j.hi for j in self.joints], dtype=float)),
            sphere_link=c(np.array([s.link for s in self.link_spheres], dtype=np.int32).reshape(ns)),
            sphere_local=c(np.array([s.center for s in self.link_spheres], dtype=float).reshape(ns, 3)),
            sphere_radius=c(np.array([s.radius for s in self.link_spheres], dtype=float).reshape(ns)),
            pairs=c(np.array(self.self_collision_pairs, dtype=np.int32).reshape(npair, 2)),
            ee_link=int(self.ee_link),
        )

    def check_q(self, q) -> np.ndarray:
        q = np.asarray(q, dtype=float)
        if q.shape != (self.n,):
            raise ValueError(f"configuration has shape {q.shape}, expected ({self.n},)")
        return q


@dataclass(frozen=True)
class FrameSet:
    """Per-link world transforms [r00..r22, px, py, pz] and the EE pose."""

    transforms: np.ndarray     # (n, 12)
    ee_position: np.ndarray    # (3,)
    ee_quaternion: np.ndarray  # (4,) w >= 0
    q: np.ndarray

    def rotation(self, link: int) -> np.ndarray:
        return self.transforms[link, :9].reshape(3, 3)

    def translation(self, link: int) -> np.ndarray:
        return self.transforms[link, 9:]


def forward_kinematics(model: RobotModel, q) -> FrameSet:
    """Device FK (FP32 chain, NVRTC-specialised for ``model``)."""
    from . import kernels
    q = model.check_q(q)
    out = kernels.fk_batch(model, q[None, :])
    return FrameSet(transforms=out["frames"][0], ee_position=out["ee"][0, :3],
                    ee_quaternion=out["ee"][0, 3:], q=q)


def collision_spheres_world(model: RobotModel, frames: FrameSet) -> list:
    from . import kernels
    sph = kernels.fk_batch(model, frames.q[None, :])["spheres"][0]
    return [Sphere(row[:3], row[3]) for row in sph]


def geometric_jacobian(model: RobotModel, q, point) -> np.ndarray:
    """6 x n point Jacobian (linear rows, then angular) from the device
    chain's world joint axes and origins."""
    from . import kernels
    q = model.check_q(q)
    point = np.asarray(point, dtype=float)
    if point.shape != (3,):
        raise ValueError("point must be a 3-vector")
    out = kernels.fk_batch(model, q[None, :])
    axes, orgs = out["axes"][0], out["origins"][0]
    rev = model.packed.jtypes == 0
    jac = np.zeros((6, model.n))
    jac[:3, rev] = np.cross(axes[rev], point - orgs[rev]).T
    jac[3:, rev] = axes[rev].T
    jac[:3, ~rev] = axes[~rev].T
    return jac


def clamp_to_limits(model: RobotModel, q) -> np.ndarray:
    q = model.check_q(q)
    p = model.packed
    return np.clip(q, p.lo, p.hi)
