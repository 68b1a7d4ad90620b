"""Summarise ncu captures in gpurun_out/ into profiles/<tag>_*.{md,json}."""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / inst"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local-load sectors"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return None


lines = [f"# ncu summary ({TAG}) -- B200, `ncu --set full --clock-control none`", ""]
traffic = {}
for kern, rep in (("cp_plan_kernel", f"prof_plan_{TAG}.ncu-rep"), ("cp_validate_kernel", f"prof_cc_{TAG}.ncu-rep"),
                  ("cp_validate_cull_kernel", f"prof_cull_{TAG}.ncu-rep"),
                  ("cp_nearest_kernel", f"prof_nn_{TAG}.ncu-rep")):
    path = os.path.join(G, rep)
    if not os.path.exists(path):
        continue
    r = raw(path)
    lines += [f"## {kern}", "", "| metric | value | unit |", "|---|---|---|"]
    for key, name in METRICS:
        if key in r:
            lines.append(f"| {name} (`{key}`) | {r[key][0]} | {r[key][1]} |")
    stalls = sorted(((k, num(v[0]) or 0) for k, v in r.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")),
                    key=lambda kv: -kv[1])[:6]
    lines += ["", "top stall reasons (pc samples): " + ", ".join(f"{k.split('stalled_')[1]} {int(v)}" for k, v in stalls), ""]
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def nbytes(key):
        v, u = r.get(key, ("0", "byte"))
        return (num(v) or 0) * units.get(u, 1)
    traffic[kern] = {"dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
                     "duration": r.get("gpu__time_duration.sum")}
lc = os.path.join(G, f"launches_{TAG}.csv")
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            d[r[ki]].append(num(r[vi]) or 0.0)
    tot = sum(sum(v) for v in d.values())
    lines += ["## launch list (`--metrics gpu__time_duration.sum`, bench.py --steps 1 --warmup 1 --queries 5)", "",
              "| kernel | launches | total time (ns) | share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v):.0f} | {100 * sum(v) / tot:.2f} % |")
    lines.append("")
with open(os.path.join(P, f"{TAG}_ncu_summary.md"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
with open(os.path.join(P, f"{TAG}_traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)
b = os.path.join(G, f"bench_{TAG}.json")
if os.path.exists(b):
    with open(b) as fh, open(os.path.join(P, f"{TAG}_bench.json"), "w") as out:
        out.write(fh.read())
print("\n".join(lines))
