"""Digest of an ncu_capture.sh result: headline metrics, instruction mix, hottest SASS lines."""
import collections
import csv
import gzip
import sys

name = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy"]
rows = list(csv.reader(open(f"gpurun_out/{name}_details.csv")))
idx = {h: i for i, h in enumerate(rows[0])}
seen = set()
for r in rows[1:]:
    mn = r[idx["Metric Name"]]
    if mn in KEEP and mn not in seen:
        seen.add(mn)
        print(f"  {mn:40s} {r[idx['Metric Value']]:>12s} {r[idx['Metric Unit']]}")
rows = list(csv.reader(gzip.open(f"gpurun_out/{name}_source.csv.gz", "rt")))
tot = 0
byop = collections.Counter()
stall = collections.Counter()
lines = []
for r in rows[2:]:
    try:
        ie, st = int(r[5]), int(r[2])
    except (ValueError, IndexError):
        continue
    t = r[1].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    tot += ie
    byop[op] += ie
    stall[op] += st
    lines.append((st, ie, r[0][-5:], r[1].strip()))
print("warp instructions", tot)
for op, c in byop.most_common(14):
    print(f"  {op:10s} {c:12d} {c / max(tot, 1) * 100:5.1f}%  stall {stall[op]}")
lines.sort(reverse=True)
for l in lines[:top]:
    print("   ", l)
