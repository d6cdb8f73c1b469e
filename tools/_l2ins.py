import sys; sys.path.insert(0, '.')
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig
L2S = int(sys.argv[1]) if len(sys.argv) > 1 else 22
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = FilterConfig(bucket_count=(1 << L2S) // B, bucket_slots=B, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda"); g.manual_seed(0)
pos = torch.randint(0, 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)
f = CuckooFilter(cfg)
for _ in range(3):
    f.clear(); r = f.insert_batch(pos)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
best = 9
for _ in range(5):
    f.clear(); torch.cuda.synchronize(); s.record(); r = f.insert_batch(pos); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print(L2S, B, "insert ms", best, n / best / 1e6, "G/s", f.last_schedule, r.n_failed, r._ctr.cpu().tolist())
