# e2e tail experiment: 2^28-slot table prefilled to (0.95*2^28 - 4Mi) keys, then a 4 Mi-key device insert (direct path)
import sys; sys.path.insert(0, '.')
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig
cfg = FilterConfig(bucket_count=1 << 24, eviction="bfs")
n = int(0.95 * cfg.total_slots); T = 1 << 22
g = torch.Generator(device="cuda"); g.manual_seed(0)
pos = torch.randint(0, 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)
f = CuckooFilter(cfg)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
best = 1e9
for _ in range(4):
    f.clear(); f.insert_batch(pos[: n - T]); torch.cuda.synchronize()
    s.record(); r = f.insert_batch(pos[n - T:]); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("tail insert ms", round(best, 3), f.last_schedule, r.n_failed, r._ctr.cpu().tolist())
