"""Summarise an ncu report: key metrics + stall reasons + hottest SASS lines."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(page, extra=()):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                       text=True)
    return r.stdout


det = list(csv.reader(io.StringIO(run("details"))))
h = det[0]
want = {"Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Grid Size",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Eligible Warps Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block",
        "SM Frequency", "DRAM Frequency"}
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run("raw"))))
if len(raw) > 2:
    hh = raw[0]
    vals = raw[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
        if k in hh:
            print(f"{k:60s} {vals[hh.index(k)]:>16s} {raw[1][hh.index(k)]}")
src = list(csv.reader(io.StringIO(run("source", ["--print-source", "sass"]))))
h = src[1]
data = src[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
for r in data:
    for c in cols:
        try:
            tot[c] += int(r[h.index(c)])
        except ValueError:
            pass
S = sum(tot.values())
print("stall reasons:", ", ".join(f"{k[6:]}={v * 100 / S:.1f}%" for k, v in tot.most_common(10)))
print("top SASS by samples:")
for r in sorted(data, key=lambda r: -int(r[iS]))[:top]:
    print(f"  {r[0][-6:]} {int(r[iS]):6d} {int(r[iE]):10d}  {r[1][:90]}")
