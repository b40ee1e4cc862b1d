"""Attribute ncu per-SASS samples to source lines via nvdisasm line info.

usage: ncu_lines.py <report.ncu-rep> <cubin> <mangled kernel name substring> [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split by function
cur_fn = None
loc = None
off2line = {}
for line in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        cur_fn = m.group(1)
        continue
    if cur_fn is None or kname not in cur_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        loc = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and loc:
        off2line[int(m.group(1), 16)] = loc
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
base = min(int(r[0], 16) for r in data)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in data:
    off = int(r[0], 16) - base
    key = off2line.get(off, ("?", 0))
    a = agg[key]
    a[0] += int(r[iS])
    a[1] += int(r[iE])
    for c in cols:
        try:
            a[2][c] += int(r[h.index(c)])
        except ValueError:
            pass
tot = sum(a[0] for a in agg.values())
print(f"total samples {tot}, mapped lines {len(agg)}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = ", ".join(f"{c[6:]}={v}" for c, v in a[2].most_common(3))
    print(f"{k[0]:14s}:{k[1]:5d}  samples {a[0]:6d} ({a[0] * 100 / tot:4.1f}%)  inst {a[1]:10d}  {reasons}")
