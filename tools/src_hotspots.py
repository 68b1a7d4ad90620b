"""Aggregate ncu source-page stall samples (cuda,sass view) per CUDA line and
per device function.  Usage: src_hotspots.py <report.ncu-rep> <source.cu>"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, srcf = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ci = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
per_line = defaultdict(lambda: [0, 0])
for r in rows[hi + 1:]:
    if len(r) <= ci or not r[0].strip().isdigit():
        continue
    ln = int(r[0])
    try:
        per_line[ln][0] += float(r[ci] or 0)
        per_line[ln][1] += float(r[ii] or 0)
    except ValueError:
        pass
src = open(srcf).read().splitlines()
# function extents: a line opening a __device__/__global__ definition
fn_at = {}
cur = "<prelude>"
pat = re.compile(r"(?:__device__|__global__)[^;(]*?\b(\w+)\s*\(")
for i, line in enumerate(src, 1):
    m = pat.search(line)
    if m and not line.strip().startswith("//") and "(" in line and not line.rstrip().endswith(";"):
        cur = m.group(1)
    fn_at[i] = cur
tot = sum(v[0] for v in per_line.values()) or 1
per_fn = defaultdict(lambda: [0, 0])
for ln, (s, n) in per_line.items():
    per_fn[fn_at.get(ln, "?")][0] += s
    per_fn[fn_at.get(ln, "?")][1] += n
print(f"total samples {tot:.0f}")
print("== per function ==")
for f, (s, n) in sorted(per_fn.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{100 * s / tot:6.2f}%  {s:8.0f}  inst {n:12.0f}  {f}")
print("== top lines ==")
for ln, (s, n) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{100 * s / tot:6.2f}%  L{ln:5d} [{fn_at.get(ln, '?')}] {src[ln - 1].strip()[:110] if ln <= len(src) else ''}")
