import sys, time, cProfile, pstats; sys.path.insert(0, '.')
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig
cfg = FilterConfig(bucket_count=1 << 18, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda"); g.manual_seed(0)
pos = torch.randint(0, 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)
f = CuckooFilter(cfg)
for _ in range(5):
    f.clear(); f.insert_batch(pos); f.delete_batch(pos)
torch.cuda.synchronize()
hs = []
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
for _ in range(20):
    f.clear(); torch.cuda.synchronize()
    s.record(); t = time.perf_counter(); r = f.insert_batch(pos); hs.append(time.perf_counter() - t); e.record()
    torch.cuda.synchronize()
print("host enqueue us: min %.1f med %.1f" % (1e6 * min(hs), 1e6 * sorted(hs)[10]), "gpu ms", s.elapsed_time(e))
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    r = f.insert_batch(pos[:1000])
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
