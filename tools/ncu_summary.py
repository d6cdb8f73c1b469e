"""Summarise an ncu --csv launch list: per launch, kernel short name, time, DRAM bytes."""
import csv
import re
import sys

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
agg = {}
order = []
for r in rows:
    k = r["ID"]
    if k not in agg:
        name = r["Kernel Name"]
        m = re.search(r"ckf::(\w+)", name)
        short = m.group(1) if m else name.split("(")[0][:40]
        tm = re.search(r"<(.*?)>\(", name)
        agg[k] = {"name": short, "tmpl": (tm.group(1)[:40] if tm and m else ""), "grid": r["Grid Size"]}
        order.append(k)
    agg[k][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = 0.0
for k in order:
    a = agg[k]
    t = a.get("gpu__time_duration.sum", 0) / 1e6
    tot += t
    rd = a.get("dram__bytes_read.sum", 0) / 1e6
    wr = a.get("dram__bytes_write.sum", 0) / 1e6
    hit = a.get("lts__t_sector_hit_rate.pct", float("nan"))
    print(f"{k:>4} {a['name']:<28} {a['tmpl']:<14} grid={a['grid']:<16} {t:8.3f} ms  rd {rd:9.1f} MB  wr {wr:9.1f} MB  L2hit {hit:5.1f}%")
print(f"total {tot:.3f} ms")
