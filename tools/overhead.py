"""Split the e2e planning time into Python, C-ABI and device parts."""
import os, sys, time, ctypes as C
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import fixtures as fx
from paper_2505_06791_b200 import _lib, kernels
from paper_2505_06791_b200.planner import PlanParams, PlanProblem, plan, prepare, _params_struct, DeviceOptions, _bind
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
p = fx.pairs()
feas = np.nonzero(fx.upright_feasible())[0][:20]
probs = [PlanProblem(m, sc, sp, p["upright_start"][k], p["upright_goal"][k], PlanParams(width=16, max_iterations=10**6, seed_offset=int(k))) for k in feas]
ctx = prepare(probs[0])
for pr in probs[:5]: plan(pr)
walls, devs, cwall, kerns = [], [], [], []
for pr in probs * 3:
    t0 = time.perf_counter(); r = plan(pr); walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(ctx.last_timing()[0]); kerns.append(ctx.last_timing()[1])
prm = _params_struct(probs[0].params, DeviceOptions())
res = (_lib.Result * 1)(); paths = np.empty((1, 1024, 7)); src = np.empty((1, 1024), np.int32)
for pr in probs * 3:
    s = np.ascontiguousarray(pr.start[None]); g = np.ascontiguousarray(pr.goal[None]); seed = np.array([1], np.int64)
    t0 = time.perf_counter()
    ctx.L.cprrtc_plan(ctx.h, C.byref(prm), 1, _lib.ptr(s), _lib.ptr(g), _lib.ptr(seed, _lib._lp), res, _lib.ptr(paths), _lib.ptr(src, _lib._ip))
    cwall.append((time.perf_counter() - t0) * 1e3 - ctx.last_timing()[0])
t0 = time.perf_counter()
for _ in range(200): _bind(probs[0], DeviceOptions())
bind_us = (time.perf_counter() - t0) / 200 * 1e6
print(f"plan() wall median {np.median(walls):.3f} ms, device {np.median(devs):.3f} ms, "
      f"host overhead {np.median(np.array(walls) - np.array(devs)) * 1e3:.0f} us; "
      f"C-ABI call overhead {np.median(cwall) * 1e3:.0f} us; _bind {bind_us:.0f} us; "
      f"device time outside the plan kernel {np.median(np.array(devs) - np.array(kerns)) * 1e3:.1f} us")
