import sys, time; sys.path[:0]=['.','tests']
import numpy as np, bench, fixtures as fx
from paper_2505_06791_b200.planner import PlanParams, PlanStream, plan_many
m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
prm = PlanParams(width=16, max_iterations=300)
for depth in (1, 2, 3, 4):
    st = PlanStream(m, sc, sp, prm, depth=depth)
    for w in range(3): st.result(st.submit(*bench.batch_arrays(w)))
    K = 16
    t0 = time.perf_counter()
    tk = [st.submit(*bench.batch_arrays(100 + k)) for k in range(min(depth, K))]
    for k in range(K):
        st.result(tk[k])
        if k + depth < K: tk.append(st.submit(*bench.batch_arrays(100 + k + depth)))
    dt = time.perf_counter() - t0
    print(f"depth {depth}: {K * 1024 / dt / 1e6:.3f} M queries/s e2e ({dt / K * 1e3:.3f} ms per batch)")
