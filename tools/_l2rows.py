import sys, json; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from paper_rows import run
from paper_2603_15486_b200 import FilterConfig
for pol, m in (("xor", 1 << 18), ("offset", 262_139)):
    r = run(FilterConfig(bucket_count=m, policy=pol, eviction="bfs", seed=0), reps=5)
    print(pol, json.dumps(r["G_ops_s"]), json.dumps(r["ms"]))
