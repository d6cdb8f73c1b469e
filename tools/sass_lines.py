"""Per-source-line instruction counts of one kernel from an ncu SASS source page.

    python tools/sass_lines.py <ncu source csv(.gz)> <cubin> [top]

ncu's CSV source page is SASS-only; this maps each SASS instruction (by its
offset in the function) to its CUDA file:line with `nvdisasm -g` on the same
cubin (-lineinfo build) and sums warp instructions executed and stall samples
per line.  The cubin must be the one that was profiled (cuobjdump -xelf all).
"""
import collections
import csv
import gzip
import re
import subprocess
import sys

src, cubin = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
op = gzip.open if src.endswith(".gz") else open
rows = list(csv.reader(op(src, "rt")))
kname = rows[0][1]
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
sass = []
for r in rows[2:]:
    try:
        sass.append((int(r[ci["Address"]], 16), r[ci["Source"]].strip(), int(r[ci["Instructions Executed"]] or 0),
                     int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)))
    except (ValueError, IndexError):
        continue
base = sass[0][0]

# mangled name: find the function in the cubin whose SASS matches in length
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*\.text\.(\S+):\n", dis)
# funcs = [pre, name1, body1, name2, body2, ...]
cands = []
for i in range(1, len(funcs) - 1, 2):
    name, body = funcs[i], funcs[i + 1]
    n_ins = len(re.findall(r"/\*[0-9a-f]{4,}\*/", body))
    cands.append((name, body, n_ins))
want = len(sass)
short = re.search(r"ckf::(\w+)<([^>]*)>", kname)
targs = ""
if short:
    vals = [re.sub(r"\(\w+\)", "", a).strip() for a in short.group(2).split(",")]
    targs = "I" + "".join(f"Li{v}E" for v in vals) + "E"
pick = None
for name, body, n_ins in cands:
    if short and f"{len(short.group(1))}{short.group(1)}{targs}" in name and abs(n_ins - want) <= 2:
        pick = (name, body)
        break
if pick is None:
    sys.exit(f"no function of {want} instructions matching {kname[:80]}")
line_of = {}
cur = "?"
for ln in pick[1].splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
stall = collections.Counter()
tot = 0
for addr, s, ie, st in sass:
    key = line_of.get(addr - base, "?")
    agg[key] += ie
    stall[key] += st
    tot += ie
print(kname[:120])
print(f"warp instructions {tot}")
for k, v in agg.most_common(top):
    print(f"  {k:28s} {v:12d} {100 * v / tot:5.1f}%  stall {stall[k]}")
