"""configs[4] throughput vs the batch's team count (isolated batches and a
PlanStream of 16 batches).  Usage: batch_teams.py T1 T2 ... (0 = every resident team)"""
import sys, time
sys.path[:0] = ['.', 'tests']
import numpy as np  # noqa: E402
import bench, fixtures as fx  # noqa: E402
from paper_2505_06791_b200 import kernels  # noqa: E402
from paper_2505_06791_b200.planner import DeviceOptions, PlanParams, PlanStream, plan_many  # noqa: E402
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prm = PlanParams(width=16, max_iterations=300)
for T in [int(x) for x in sys.argv[1:]]:
    opt = DeviceOptions(teams=T)
    ctx = kernels.context(m, 0)
    for w in range(3):
        plan_many(m, sc, sp, *bench.batch_arrays(w), prm, opt)
    dev = []
    for k in range(8):
        plan_many(m, sc, sp, *bench.batch_arrays(100 + k), prm, opt)
        dev.append(ctx.last_timing()[0])
    st = PlanStream(m, sc, sp, prm, opt, depth=2)
    for w in range(2):
        st.result(st.submit(*bench.batch_arrays(w)))
    K = 16
    t0 = time.perf_counter()
    tk = [st.submit(*bench.batch_arrays(100 + k)) for k in range(2)]
    for k in range(K):
        st.result(tk[k])
        if k + 2 < K:
            tk.append(st.submit(*bench.batch_arrays(100 + k + 2)))
    dt = time.perf_counter() - t0
    print(f"teams {T}: isolated device {1024 / np.median(dev) * 1e-3:.3f} M q/s ({np.median(dev):.3f} ms); "
          f"stream e2e {K * 1024 / dt / 1e6:.3f} M q/s", flush=True)
