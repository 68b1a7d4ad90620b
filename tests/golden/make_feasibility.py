"""Which upright pairs does the reference (C oracle port) solve with a long budget?"""
import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from concurrent.futures import ProcessPoolExecutor

def job(k):
    import fixtures as fx
    from oracle import oracle as orc
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("upright")
    p = fx.pairs()
    best = None
    for seed in (0, 10000, 20000):
        r = orc.plan(m.packed, sc.packed(), sp.packed, p["upright_start"][k], p["upright_goal"][k],
                     width=16, max_iterations=10**7, time_budget_ms=20000.0, seed_offset=seed)
        if r["status"] == "Solved":
            return k, True, r["wall_ms"], r["stats"]["iterations"]
    return k, False, r["wall_ms"], r["stats"]["iterations"]

if __name__ == "__main__":
    with ProcessPoolExecutor(8) as ex:
        res = list(ex.map(job, range(100)))
    json.dump({"generated_by": "tests/golden/make_feasibility.py (C oracle, 3 seeds x 20 s)", "upright_solved_by_reference": [bool(r[1]) for r in res], "reference_wall_ms": [r[2] for r in res]}, open(os.path.join(ROOT, "tests", "golden", "upright_feasibility.json"), "w"))
    print(sum(r[1] for r in res), "solved of", len(res))
    print([r[0] for r in res if not r[1]])
