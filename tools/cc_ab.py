"""CC lockstep kernel throughput A/B (999-box shelf, 16384 motions x 16, flag off)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import fixtures as fx
from paper_2505_06791_b200 import kernels
m, sc = fx.robot("arm7"), fx.scene("shelf_x111")
B, W = 16384, 16
qs = kernels.halton_batch(m, 2 * B, 1, 12345)
t = np.linspace(0, 1, W)[None, :, None]
wps = qs[0::2][:, None, :] * (1 - t) + qs[1::2][:, None, :] * t
kernels.validate_batch(m, sc, wps[:64], False)
best = min(kernels.validate_batch(m, sc, wps, False)["kernel_ms"] for _ in range(5))
r = kernels.validate_batch(m, sc, wps, False)
print(os.environ.get("CPRRTC_SB"), os.environ.get("CPRRTC_VMINB"), f"{r['gpu_checks'].sum() / (best * 1e-3) / 1e12:.3f} T checks/s", best)
