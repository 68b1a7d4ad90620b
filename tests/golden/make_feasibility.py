"""Which pairs of a benchmark config does the reference planner (C oracle
port, reference semantics) solve with a long budget?  3 seeds x 20 s each.

  python tests/golden/make_feasibility.py            # upright Panda, 100 pairs
  python tests/golden/make_feasibility.py dense8     # configs[3]: arm8_dense line, 20 pairs
"""
import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from concurrent.futures import ProcessPoolExecutor

CFG = {
    "upright": dict(robot="arm7", scene="table", spec="upright", key="upright", n=100,
                    out="upright_feasibility.json", field="upright_solved_by_reference"),
    "dense8": dict(robot="arm8_dense", scene="table", spec="table_line_8", key="dense8_line", n=20,
                   out="dense8_feasibility.json", field="dense8_line_solved_by_reference"),
}


def job(args):
    name, k = args
    c = CFG[name]
    import fixtures as fx
    from oracle import oracle as orc
    m, sc, sp = fx.robot(c["robot"]), fx.scene(c["scene"]), fx.spec(c["spec"])
    p = fx.pairs()
    for seed in (0, 10000, 20000):
        r = orc.plan(m.packed, sc.packed(), sp.packed, p[c["key"] + "_start"][k], p[c["key"] + "_goal"][k],
                     width=16, max_iterations=10**7, time_budget_ms=20000.0, seed_offset=seed)
        if r["status"] == "Solved":
            return k, True, r["wall_ms"], r["stats"]["iterations"]
    return k, False, r["wall_ms"], r["stats"]["iterations"]


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "upright"
    c = CFG[name]
    n = min(c["n"], len(__import__("fixtures").pairs()[c["key"] + "_seed"]))
    with ProcessPoolExecutor(8) as ex:
        res = list(ex.map(job, [(name, k) for k in range(n)]))
    json.dump({"generated_by": f"tests/golden/make_feasibility.py {name} (C oracle, 3 seeds x 20 s)",
               c["field"]: [bool(r[1]) for r in res], "reference_wall_ms": [r[2] for r in res]},
              open(os.path.join(ROOT, "tests", "golden", c["out"]), "w"))
    print(sum(r[1] for r in res), "solved of", len(res))
    print([r[0] for r in res if not r[1]])
