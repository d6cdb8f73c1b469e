import sys; sys.path.insert(0, ".")
import torch, numpy as np
from paper_2603_15486_b200 import CuckooFilter, FilterConfig
from paper_2603_15486_b200.bench_harness import gen_keys, _dev
cfg = FilterConfig(bucket_count=(1 << 26) // 16, fingerprint_bits=8, bucket_slots=16, eviction="bfs")
filt = CuckooFilter(cfg)
n = int(0.95 * cfg.total_slots)
filt.insert_batch(_dev(gen_keys(n, 0)))
probe = _dev(gen_keys(100_000_000, 0, negative=True))
for _ in range(2):
    h = filt.query_batch(probe)
torch.cuda.synchronize()
print(float(h.float().mean()))
