"""Run one op of the bench config a few times (target for ncu --set full)."""
import os
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

op = sys.argv[1] if len(sys.argv) > 1 else "query"
tiled = {"auto": None, "on": True, "off": False}[sys.argv[2] if len(sys.argv) > 2 else "auto"]
log2 = int(os.environ.get("LOG2", 28))
cfg = FilterConfig(bucket_count=(1 << log2) // 16, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda")
g.manual_seed(0)
pos = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64, generator=g)
filt = CuckooFilter(cfg, tiled=tiled)
filt.insert_batch(pos)
for _ in range(2):
    if op == "query":
        filt.query_batch(pos)
    elif op == "insert":
        filt.clear()
        filt.insert_batch(pos)
    elif op == "delete":
        filt.delete_batch(pos)
        filt.insert_batch(pos)
torch.cuda.synchronize()
print("done", op)
