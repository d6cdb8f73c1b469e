"""Insert 95% then query disjoint negatives twice (ncu target for the lookup- path)."""
import os
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

log2 = int(os.environ.get("LOG2", 28))
cfg = FilterConfig(bucket_count=(1 << log2) // 16, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda")
g.manual_seed(0)
pos = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64, generator=g)
neg = torch.randint(1 << 32, 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)
filt = CuckooFilter(cfg)
filt.insert_batch(pos)
for _ in range(2):
    filt.query_batch(neg)
torch.cuda.synchronize()
print("done", filt.last_counters())
