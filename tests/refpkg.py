"""The reference package itself (``maniplan``, stock build in oracle/_ref by
oracle/build_ref.sh) for tests and bench.py's CPU arms.  TEST / BASELINE
INFRASTRUCTURE ONLY: the product never imports it.

* ``load(kernels)`` imports it with ``MANIPLAN_KERNELS`` = ``compiled`` (the
  reference's FP64 Cython backend) or ``b200`` -- the two-line selector
  patch of INTEGRATION.md section 1 (``maniplan/_kernels/__init__.py:33-44``),
  applied by rebinding ``active`` / ``active_name`` and every module's ``_K``
  (the reference modules bind ``from ._kernels import active as _K`` at
  import: ``constraints.py:20``, ``kinematics.py:37``, ``projection.py:28``,
  ``validation.py:24``), which is exactly what the patched selector yields.
  A process holds one choice; tests that need ``b200`` run in a subprocess.
* ``to_ref_*`` rebuild this repo's model / scene / spec objects (which carry
  the reference's fields) as the reference's own dataclasses.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def available() -> bool:
    return os.path.exists(os.path.join(REF, "maniplan", "planner.refpyc"))


def _ref_path_hook(path):
    """Finder for oracle/_ref only: the reference's own bytecode (sourceless,
    suffix .refpyc -- see oracle/build_ref.sh) and its compiled extension."""
    import importlib.machinery as im
    if not os.path.abspath(path).startswith(REF):
        raise ImportError("not oracle/_ref")
    return im.FileFinder(path, (im.ExtensionFileLoader, im.EXTENSION_SUFFIXES),
                         (im.SourcelessFileLoader, [".refpyc"]))


def load(kernels: str = "compiled"):
    if not available():
        raise RuntimeError("oracle/_ref is not built (oracle/build_ref.sh)")
    if _ref_path_hook not in sys.path_hooks:
        sys.path_hooks.insert(0, _ref_path_hook)
        sys.path_importer_cache.clear()
    if REF not in sys.path:
        sys.path.insert(0, REF)
    if kernels == "b200":
        os.environ["MANIPLAN_KERNELS"] = "compiled"
        import maniplan
        from maniplan import _kernels, constraints, kinematics, projection, validation

        from paper_2505_06791_b200 import kernels as b200
        _kernels.active = b200
        _kernels.active_name = b200.name
        maniplan.kernel_backend = b200.name
        for mod in (constraints, kinematics, projection, validation):
            mod._K = b200
        return maniplan
    os.environ["MANIPLAN_KERNELS"] = kernels
    import maniplan
    if maniplan.kernel_backend != "compiled" and kernels == "compiled":
        raise RuntimeError(f"reference backend is {maniplan.kernel_backend!r}, not compiled")
    return maniplan


def to_ref_robot(M, model):
    from maniplan.kinematics import Joint, LinkSphere, RobotModel
    return RobotModel(
        joints=tuple(Joint(j.jtype, j.axis, j.origin_xyz, j.origin_rpy, j.lo, j.hi, j.name)
                     for j in model.joints),
        link_spheres=tuple(LinkSphere(s.link, s.center, s.radius) for s in model.link_spheres),
        ee_link=model.ee_link, self_collision_pairs=tuple(tuple(p) for p in model.self_collision_pairs),
        name=model.name, zero_pose_ee=model.zero_pose_ee)


def to_ref_scene(M, scene):
    from maniplan.geometry import Aabb, Scene, Sphere
    return Scene(boxes=tuple(Aabb(b.min, b.max) for b in scene.boxes),
                 spheres=tuple(Sphere(s.center, s.radius) for s in scene.spheres), name=scene.name)


def to_ref_spec(M, spec):
    if spec is None:
        return None
    from maniplan.constraints import ConstraintSpec, LineConstraint, PlaneConstraint
    p = spec.position
    if hasattr(p, "normal"):
        pos = PlaneConstraint(p.normal, p.offset)
    else:
        pos = LineConstraint(p.point, p.direction, basis=getattr(p, "basis", None))
    return ConstraintSpec(pos, fixed_orientation=spec.fixed_orientation,
                          angular_weight=spec.angular_weight, tau_task=spec.tau_task)


def to_ref_problem(M, prob, cache=None):
    """The reference PlanProblem of one of ours (model/scene/spec converted
    once per object when ``cache`` is a dict)."""
    cache = {} if cache is None else cache

    def conv(obj, fn):
        if obj is None:
            return None
        key = (fn.__name__, id(obj))
        hit = cache.get(key)
        if hit is None or hit[0] is not obj:
            hit = cache[key] = (obj, fn(M, obj))
        return hit[1]

    p = prob.params
    pp = p.projection
    proj = M.ProjectionParams(alpha=pp.alpha, max_iters=pp.max_iters, lam=pp.lam,
                              tau_task=pp.tau_task, tau_sm=pp.tau_sm)
    params = M.PlanParams(step_size=p.step_size, width=p.width, projection=proj,
                          max_iterations=p.max_iterations,
                          time_budget_ms=p.time_budget_ms, connect_tolerance=p.connect_tolerance,
                          projection_mode=p.projection_mode, flag_mode=p.flag_mode,
                          seed_offset=p.seed_offset, deterministic=p.deterministic,
                          attempts=p.attempts, max_connect_segments=p.max_connect_segments)
    return M.PlanProblem(conv(prob.model, to_ref_robot), conv(prob.scene, to_ref_scene),
                         conv(prob.spec, to_ref_spec), prob.start, prob.goal, params, prob.name)
