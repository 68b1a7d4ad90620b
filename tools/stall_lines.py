"""Attribute an ncu capture's stall samples and local-memory traffic to CUDA
source lines and device functions (the ``--page source --print-source
cuda,sass`` view of a ``--set full --import-source on`` report).

Usage: stall_lines.py <report.ncu-rep> <source.cu> [top]
Prints, per function and per line: all stall samples, long-scoreboard
samples, executed instructions and executed local loads / stores (LDL/STL,
the stack frame and spilled / dynamically indexed arrays)."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, srcf = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
c_all = h.index("Warp Stall Sampling (All Samples)")
c_lsb = h.index("stall_long_sb")
c_ins = h.index("Instructions Executed")
F = ("samples", "long_sb", "inst", "ldl", "stl")
per_line = defaultdict(lambda: dict.fromkeys(F, 0.0))


def num(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


line = None
for r in rows[hi + 1:]:
    if len(r) <= c_lsb:
        continue
    if r[0].strip().isdigit():          # a CUDA source line: its aggregate
        line = int(r[0])
        d = per_line[line]
        d["samples"] += num(r[c_all])
        d["long_sb"] += num(r[c_lsb])
        d["inst"] += num(r[c_ins])
        continue
    if line is None:                    # SASS rows of the current line
        continue
    op = r[3].split()
    op = [t for t in op if not t.startswith("@")]
    if op and op[0].startswith("LDL"):
        per_line[line]["ldl"] += num(r[c_ins])
    elif op and op[0].startswith("STL"):
        per_line[line]["stl"] += num(r[c_ins])

src = open(srcf).read().splitlines()
fn_at, cur = {}, "<prelude>"
pat = re.compile(r"(?:__device__|__global__)[^;(]*?\b(\w+)\s*\(")
for i, text in enumerate(src, 1):
    m = pat.search(text)
    if m and not text.strip().startswith("//") and not text.rstrip().endswith(";"):
        cur = m.group(1)
    fn_at[i] = cur
tot = {k: sum(d[k] for d in per_line.values()) or 1.0 for k in F}
per_fn = defaultdict(lambda: dict.fromkeys(F, 0.0))
for ln, d in per_line.items():
    for k in F:
        per_fn[fn_at.get(ln, "?")][k] += d[k]
print(f"totals: samples {tot['samples']:.0f}, long_scoreboard {tot['long_sb']:.0f}, "
      f"instructions {tot['inst']:.0f}, local loads {tot['ldl']:.0f}, local stores {tot['stl']:.0f} (warp-level)")
hdr = f"{'samples%':>9} {'long_sb%':>9} {'LDL':>9} {'STL':>9}  "
print("\n== per function (by samples) ==\n" + hdr + "function")
for f, d in sorted(per_fn.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    print(f"{100 * d['samples'] / tot['samples']:9.2f} {100 * d['long_sb'] / tot['long_sb']:9.2f} "
          f"{d['ldl']:9.0f} {d['stl']:9.0f}  {f}")
print("\n== lines by long-scoreboard samples ==\n" + hdr + "line")
for ln, d in sorted(per_line.items(), key=lambda kv: -kv[1]["long_sb"])[:top]:
    print(f"{100 * d['samples'] / tot['samples']:9.2f} {100 * d['long_sb'] / tot['long_sb']:9.2f} "
          f"{d['ldl']:9.0f} {d['stl']:9.0f}  L{ln} [{fn_at.get(ln, '?')}] "
          f"{src[ln - 1].strip()[:90] if ln <= len(src) else ''}")
print("\n== lines by local memory instructions executed ==\n" + hdr + "line")
for ln, d in sorted(per_line.items(), key=lambda kv: -(kv[1]["ldl"] + kv[1]["stl"]))[:top]:
    if d["ldl"] + d["stl"] == 0:
        break
    print(f"{100 * d['samples'] / tot['samples']:9.2f} {100 * d['long_sb'] / tot['long_sb']:9.2f} "
          f"{d['ldl']:9.0f} {d['stl']:9.0f}  L{ln} [{fn_at.get(ln, '?')}] "
          f"{src[ln - 1].strip()[:90] if ln <= len(src) else ''}")
