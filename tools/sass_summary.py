"""Resource usage and SASS instruction mix of the NVRTC modules (the robot-
specialised planner and parity kernels), from the cached sm_100a cubins:
registers / stack / shared per kernel (cuobjdump -res-usage, the ptxas -v
figures) and per-kernel counts of the instruction classes that matter here
(packed FP32x2, FP32 pipe, MUFU, local memory, shared / global loads,
barriers, calls).  Usage: sass_summary.py [robot G kind orient parity]..."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import fixtures as fx  # noqa: E402
from paper_2505_06791_b200 import _lib  # noqa: E402

MODS = [("arm7", 16, 0, 1, 0), ("arm7", 16, 0, 0, 1)]
if len(sys.argv) > 1:
    a = sys.argv[1:]
    MODS = [(a[i], int(a[i + 1]), int(a[i + 2]), int(a[i + 3]), int(a[i + 4])) for i in range(0, len(a), 5)]
KEEP = {"cp_plan_kernel", "cp_validate_kernel", "cp_validate_cull_kernel", "cp_nearest_kernel", "cp_project_kernel",
        "cp_dense_kernel", "cp_check_kernel"}
CLASSES = ["FFMA", "FFMA2", "FADD", "FADD2", "FMUL", "FMUL2", "FMNMX", "FMNMX3", "FSETP", "MUFU", "LDL", "STL", "LDS",
           "LDG", "STG", "SHFL", "BAR", "CALL"]

for name, G, kind, orient, parity in MODS:
    cub = _lib.precompile(fx.robot(name).packed, G, kind, orient, parity)
    res = subprocess.run(["cuobjdump", "-res-usage", cub], capture_output=True, text=True).stdout
    sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
    usage = {}
    fn = None
    for line in res.splitlines():
        m = re.search(r"Function (\w+):", line)
        if m:
            fn = m.group(1)
        elif fn and "REG:" in line:
            usage[fn] = " ".join(line.split()[:5])
    cnt = collections.defaultdict(collections.Counter)
    fn = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", line)
        if m and fn:
            cnt[fn][m.group(1)] += 1
            cnt[fn]["total"] += 1
    print(f"## {name} G{G} kind{kind} orient{orient} {'parity' if parity else 'plan'} module "
          f"({os.path.basename(cub)})\n")
    print("| kernel | resources | SASS | " + " | ".join(CLASSES) + " |")
    print("|---|---|---|" + "---|" * len(CLASSES))
    for f in sorted(cnt):
        if f not in KEEP:
            continue
        c = cnt[f]
        print(f"| {f} | {usage.get(f, '')} | {c['total']} | " + " | ".join(str(c[k]) for k in CLASSES) + " |")
    print()
