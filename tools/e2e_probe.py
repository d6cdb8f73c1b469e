"""e2e (pinned host keys -> host answers) timing per op vs chunk size and path."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

cfg = FilterConfig(bucket_count=1 << 24, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(); g.manual_seed(0)
pos = torch.randint(0, 1 << 32, (n,), dtype=torch.int64, generator=g).pin_memory()
neg = torch.randint(1 << 32, 1 << 62, (n,), dtype=torch.int64, generator=g).pin_memory()

def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, r

for tiled in (None, False):
    for chunk in (1 << 24, 1 << 25, 1 << 26, 1 << 30):
        CuckooFilter.HOST_CHUNK = chunk
        f = CuckooFilter(cfg, tiled=tiled)
        for rep in range(2):
            ti, r = t(lambda: f.insert_batch(pos)); _ = r.ok
            tq, _ = t(lambda: f.query_batch(pos))
            tn, _ = t(lambda: f.query_batch(neg))
            td, _ = t(lambda: f.delete_batch(pos))
        print(f"tiled={tiled} chunk=2^{chunk.bit_length()-1}: insert {ti:.1f} q+ {tq:.1f} q- {tn:.1f} del {td:.1f} ms  total {ti+tq+tn+td:.1f}", flush=True)
        del f; torch.cuda.empty_cache()
