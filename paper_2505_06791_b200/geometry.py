"""World obstacles: axis-aligned boxes and spheres, their packed device layout,
clearance queries and union-preserving densification.

Public names mirror ``maniplan/geometry.py`` (Aabb, Sphere, Scene,
PackedScene, subdivide_scene ...; the YAML loaders are the reference's own).  The packed arrays have the
reference layout (``geometry.py:101-135``); the device copy is FP32 in
shared memory ("Data layout").
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Aabb", "Sphere", "Scene", "PackedScene", "sphere_aabb_clearance",
    "sphere_sphere_clearance", "subdivide_box", "subdivide_scene",
    "scene_contains", "load_scene", "dump_scene",
]


def _vec3(v, what):
    a = np.asarray(v, dtype=float)
    if a.shape != (3,):
        raise ValueError(f"{what} must be a 3-vector")
    return a


@dataclass(frozen=True)
class Aabb:
    """Closed axis-aligned box [min, max] in metres."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        lo = _vec3(self.min, "Aabb min")
        hi = _vec3(self.max, "Aabb max")
        if not (np.isfinite(lo).all() and np.isfinite(hi).all()):
            raise ValueError("Aabb corners must be finite")
        bad = np.nonzero(lo > hi)[0]
        if bad.size:
            raise ValueError(f"Aabb min > max on axis {int(bad[0])}")
        object.__setattr__(self, "min", lo)
        object.__setattr__(self, "max", hi)

    @property
    def extents(self) -> np.ndarray:
        return self.max - self.min

    @property
    def volume(self) -> float:
        ex, ey, ez = self.extents
        return float(ex * ey * ez)

    def contains(self, point) -> bool:
        p = np.asarray(point, dtype=float)
        return bool((p >= self.min).all() and (p <= self.max).all())


@dataclass(frozen=True)
class Sphere:
    center: np.ndarray
    radius: float

    def __post_init__(self):
        c = _vec3(self.center, "Sphere center")
        r = float(self.radius)
        if not (np.isfinite(c).all() and math.isfinite(r)):
            raise ValueError("Sphere must be finite")
        if r <= 0.0:
            raise ValueError("Sphere radius must be > 0")
        object.__setattr__(self, "center", c)
        object.__setattr__(self, "radius", r)


@dataclass(frozen=True)
class PackedScene:
    """Flat C-contiguous float64 arrays (reference layout)."""

    box_min: np.ndarray      # (B, 3)
    box_max: np.ndarray      # (B, 3)
    sph_center: np.ndarray   # (E, 3)
    sph_radius: np.ndarray   # (E,)

    @property
    def n_boxes(self) -> int:
        return int(self.box_min.shape[0])

    @property
    def n_spheres(self) -> int:
        return int(self.sph_center.shape[0])


@dataclass(frozen=True)
class Scene:
    """Immutable obstacle set; empty means free space."""

    boxes: tuple = ()
    spheres: tuple = ()
    name: str = ""
    _packed: PackedScene | None = field(default=None, init=False, repr=False,
                                        compare=False, hash=False)

    def __post_init__(self):
        object.__setattr__(self, "boxes", tuple(self.boxes))
        object.__setattr__(self, "spheres", tuple(self.spheres))

    @property
    def primitive_count(self) -> int:
        return len(self.boxes) + len(self.spheres)

    def packed(self) -> PackedScene:
        # Scenes are immutable, so the packing is built once (the reference
        # rebuilds it on every call, geometry.py:97-98).
        if self._packed is None:
            nb, ne = len(self.boxes), len(self.spheres)
            bmin = np.array([b.min for b in self.boxes], dtype=float).reshape(nb, 3)
            bmax = np.array([b.max for b in self.boxes], dtype=float).reshape(nb, 3)
            sc = np.array([s.center for s in self.spheres], dtype=float).reshape(ne, 3)
            sr = np.array([s.radius for s in self.spheres], dtype=float).reshape(ne)
            c = np.ascontiguousarray
            object.__setattr__(self, "_packed", PackedScene(c(bmin), c(bmax), c(sc), c(sr)))
        return self._packed


def _as_packed_scene(scene) -> PackedScene:
    p = scene.packed() if callable(getattr(scene, "packed", None)) else scene
    return p


def sphere_aabb_clearance(s: Sphere, b: Aabb) -> float:
    """Centre-to-box distance minus radius (negative iff overlapping).

    Evaluated on the device (FP32, the planner's arithmetic); see
    ``clearances_batch`` for the vectorised form.
    """
    from . import kernels
    return float(kernels.clearance_batch(
        np.array([[*s.center, s.radius]]),
        np.array([[*b.min, *b.max]]), kind="box")[0])


def sphere_sphere_clearance(a: Sphere, b: Sphere) -> float:
    """Centre distance minus both radii (negative iff overlapping); device."""
    from . import kernels
    return float(kernels.clearance_batch(
        np.array([[*a.center, a.radius]]),
        np.array([[*b.center, b.radius]]), kind="sphere")[0])


def scene_contains(scene: Scene, point) -> bool:
    """True iff the point lies in any (closed) primitive."""
    p = np.asarray(point, dtype=float)
    if any(b.contains(p) for b in scene.boxes):
        return True
    for s in scene.spheres:
        d = p - s.center
        if float(d @ d) <= s.radius * s.radius:
            return True
    return False


def subdivide_box(box: Aabb, factor: int) -> list:
    """``factor`` boxes tiling ``box`` exactly, by the reference's
    densification rule (geometry.py:175-210): the largest-volume piece
    (first on ties) is cut at the midpoint of its longest axis (lowest axis on
    ties) until there are ``factor`` pieces.  Pieces are kept as (k, 3) corner
    arrays; volumes are the same e0*e1*e2 products, so ties break identically."""
    if factor < 1:
        raise ValueError("subdivision factor must be >= 1")
    lo = box.min[None, :].copy()
    hi = box.max[None, :].copy()
    while lo.shape[0] < factor:
        ext = hi - lo
        k = int(np.argmax(ext[:, 0] * ext[:, 1] * ext[:, 2]))
        ax = int(np.argmax(ext[k]))
        mid = 0.5 * (lo[k, ax] + hi[k, ax])
        upper_lo = lo[k].copy()
        upper_lo[ax] = mid
        lower_hi = hi[k].copy()
        lower_hi[ax] = mid
        lo = np.insert(lo, k + 1, upper_lo, axis=0)
        hi = np.insert(hi, k + 1, hi[k], axis=0)
        hi[k] = lower_hi
    return [Aabb(a, b) for a, b in zip(lo, hi)]


def subdivide_scene(scene: Scene, factor: int) -> Scene:
    if factor < 1:
        raise ValueError("subdivision factor must be >= 1")
    if factor == 1:
        return scene
    boxes = [piece for b in scene.boxes for piece in subdivide_box(b, factor)]
    return Scene(boxes=tuple(boxes), spheres=scene.spheres,
                 name=f"{scene.name}@{factor}x" if scene.name else "")
