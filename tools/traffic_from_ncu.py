"""Per-op DRAM traffic from an ncu launch list of `bench.py --steps 1 --warmup 1 --no-e2e`.

Groups the launches of the LAST bench step (insert / lookup+ / lookup- / delete,
in that order) and writes profiles/traffic.json: bytes per op call
(dram__bytes_read.sum + dram__bytes_write.sum summed over the op's kernels)
plus the kernel list, for bench.py's roofline.traffic field.
"""
import csv
import json
import re
import sys

path, out = sys.argv[1], sys.argv[2]
rows = list(csv.DictReader([ln for ln in open(path) if ln.startswith('"')]))
launches = {}
for r in rows:
    k = int(r["ID"])
    d = launches.setdefault(k, {"name": r["Kernel Name"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
seq = [launches[k] for k in sorted(launches)]
ours = [d for d in seq if "ckf::" in d["name"]]
for d in ours:
    m = re.search(r"ckf::(\w+)<([^>]*)>", d["name"]) or re.search(r"ckf::(\w+)", d["name"])
    d["short"] = m.group(1)
    args = [a.strip() for a in m.group(2).split(",")] if m.lastindex and m.lastindex > 1 else []
    d["op"] = (int(args[0]) if args and m.group(1).startswith(("tile", "region"))
               and m.group(1) != "region_sample_kernel" else None)
    # a new op call starts at its first pass: the keys' bin kernel (region SRC_KEYS = 0) or a direct kernel
    d["start"] = (d["short"] in ("region_sample_kernel",)
                  or (d["short"] == "region_bin_kernel" and args[-1] == "0")
                  or d["short"] in ("insert_kernel", "query_kernel", "delete_kernel"))


def op_of(d):
    if d["short"] in ("insert_kernel", "evict_kernel", "evict_bfs_kernel"):
        return "insert"
    if d["short"] in ("query_kernel", "region_sample_kernel"):
        return "query"
    if d["short"] == "delete_kernel":
        return "delete"
    if d["op"] is not None:
        return {0: "query", 1: "insert", 2: "delete"}[d["op"]]
    return None


groups = []
for d in ours:
    o = op_of(d)
    after_sample = bool(groups) and groups[-1][1][-1]["short"] in ("region_sample_kernel", "fill_bits_kernel")
    if (d["start"] and not after_sample) or not groups:
        groups.append((o, [d]))
    else:
        groups[-1][1].append(d)
# the bench's verification pass repeats insert, q+, q-, delete after the timed step;
# take the last four groups named insert, query, query, delete
names = ["insert", "lookup+", "lookup-", "delete"]
tail = groups[-4:]
res = {}
for nm, (o, ks) in zip(names, tail):
    res[nm] = int(sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks))
    res[nm + "_kernels"] = [(k["short"], round(k.get("gpu__time_duration.sum", 0) / 1e6, 4)) for k in ks]
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
