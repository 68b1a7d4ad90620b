"""World obstacles: axis-aligned boxes and spheres, their packed device layout,
clearance queries and union-preserving densification.

Public names mirror ``maniplan/geometry.py`` (Aabb, Sphere, Scene,
PackedScene, subdivide_scene, load_scene ...).  The packed arrays have the
reference layout (``geometry.py:101-135``); the device copy is FP32 in
shared memory ("Data layout").
"""

from __future__ import annotations

import io
import math
import os
from dataclasses import dataclass, field

import numpy as np
import yaml

from .errors import SceneFormatError

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


def _halve(box: Aabb):
    ext = box.extents
    ax = 0
    for k in (1, 2):               # longest axis, lowest index on ties
        if ext[k] > ext[ax]:
            ax = k
    cut = 0.5 * (box.min[ax] + box.max[ax])
    lo_hi = box.max.copy()
    lo_hi[ax] = cut
    hi_lo = box.min.copy()
    hi_lo[ax] = cut
    return Aabb(box.min.copy(), lo_hi), Aabb(hi_lo, box.max.copy())


def subdivide_box(box: Aabb, factor: int) -> list:
    """``factor`` boxes tiling ``box`` exactly: keep halving the largest
    piece (first on ties) -- the reference's densification rule
    (geometry.py:190-210)."""
    if factor < 1:
        raise ValueError("subdivision factor must be >= 1")
    pieces = [box]
    while len(pieces) < factor:
        vols = [p.volume for p in pieces]
        k = int(np.argmax(vols))
        pieces[k:k + 1] = list(_halve(pieces[k]))
    return pieces


def subdivide_scene(scene: Scene, factor: int) -> Scene:
    if factor < 1:
        raise ValueError("subdivision factor must be >= 1")
    if factor == 1:
        return scene
    boxes = [piece for b in scene.boxes for piece in subdivide_box(b, factor)]
    return Scene(boxes=tuple(boxes), spheres=scene.spheres,
                 name=f"{scene.name}@{factor}x" if scene.name else "")


# --------------------------------------------------------------------------
# YAML format (reference geometry.py:229-340): name / boxes[min,max] /
# spheres[center,radius]
# --------------------------------------------------------------------------

def read_source(source, err=SceneFormatError):
    """(text, where) from a path, a YAML string, bytes or a stream."""
    if hasattr(source, "read"):
        data = source.read()
        if isinstance(data, bytes):
            data = data.decode("utf-8")
        return data, getattr(source, "name", "<stream>")
    if isinstance(source, bytes):
        return source.decode("utf-8"), "<bytes>"
    if isinstance(source, str):
        if "\n" not in source and os.path.exists(source):
            with io.open(source, encoding="utf-8") as fh:
                return fh.read(), source
        return source, "<string>"
    if hasattr(source, "__fspath__"):
        with io.open(os.fspath(source), encoding="utf-8") as fh:
            return fh.read(), os.fspath(source)
    raise err(f"cannot read document from {type(source).__name__}")


def _parse_yaml(text, where, err):
    try:
        return yaml.safe_load(text)
    except yaml.YAMLError as exc:
        mark = getattr(exc, "problem_mark", None)
        raise err(f"not valid YAML: {exc}",
                  f"{where}:line {mark.line + 1}" if mark else where) from None


def _num3(v, where):
    if not isinstance(v, (list, tuple)) or len(v) != 3:
        raise SceneFormatError("expected a 3-element list", where)
    try:
        return np.array([float(x) for x in v])
    except (TypeError, ValueError):
        raise SceneFormatError("expected numeric entries", where) from None


def scene_from_dict(doc, where="scene") -> Scene:
    doc = {} if doc is None else doc
    if not isinstance(doc, dict):
        raise SceneFormatError("document root must be a mapping", where)
    extra = set(doc) - {"name", "boxes", "spheres"}
    if extra:
        raise SceneFormatError(f"unknown field {sorted(extra)[0]!r}", where)
    name = doc.get("name", "")
    if not isinstance(name, str):
        raise SceneFormatError("name must be a string", f"{where}.name")
    boxes, spheres = [], []
    for i, ent in enumerate(doc.get("boxes") or []):
        loc = f"{where}.boxes[{i}]"
        if not isinstance(ent, dict):
            raise SceneFormatError("expected a mapping with min/max", loc)
        lo, hi = _num3(ent.get("min"), f"{loc}.min"), _num3(ent.get("max"), f"{loc}.max")
        bad = np.nonzero(lo > hi)[0]
        if bad.size:
            raise SceneFormatError(f"max < min on axis {int(bad[0])}", loc)
        try:
            boxes.append(Aabb(lo, hi))
        except ValueError as exc:
            raise SceneFormatError(str(exc), loc) from None
    for i, ent in enumerate(doc.get("spheres") or []):
        loc = f"{where}.spheres[{i}]"
        if not isinstance(ent, dict):
            raise SceneFormatError("expected a mapping with center/radius", loc)
        c = _num3(ent.get("center"), f"{loc}.center")
        try:
            r = float(ent.get("radius"))
        except (TypeError, ValueError):
            raise SceneFormatError("radius must be a number", loc) from None
        try:
            spheres.append(Sphere(c, r))
        except ValueError as exc:
            raise SceneFormatError(str(exc), loc) from None
    return Scene(boxes=tuple(boxes), spheres=tuple(spheres), name=name)


def load_scene(source) -> Scene:
    text, where = read_source(source)
    return scene_from_dict(_parse_yaml(text, where, SceneFormatError), where)


def dump_scene(scene: Scene) -> str:
    return yaml.safe_dump({
        "name": scene.name,
        "boxes": [{"min": b.min.tolist(), "max": b.max.tolist()} for b in scene.boxes],
        "spheres": [{"center": s.center.tolist(), "radius": s.radius}
                    for s in scene.spheres],
    }, sort_keys=False)
