"""Small forced-region runs of insert / query / delete (compute-sanitizer target)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

for f, b, pol in [(16, 16, "xor"), (8, 16, "offset"), (16, 32, "xor")]:
    m = (1 << 11) - (3 if pol == "offset" else 0)
    cfg = FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b, policy=pol, eviction="bfs", seed=1)
    rng = np.random.default_rng(0)
    keys = rng.integers(0, 1 << 62, size=int(0.95 * cfg.total_slots), dtype=np.uint64)
    neg = rng.integers(1 << 62, 1 << 63, size=len(keys), dtype=np.uint64)
    filt = CuckooFilter(cfg, tiled=True)
    r = filt.insert_batch(keys)
    q = filt.query_batch(keys)
    qn = filt.query_batch(neg)
    d = filt.delete_batch(keys)
    torch.cuda.synchronize()
    print(f, b, pol, r.n_failed, bool(q.all()), float(qn.mean()), int(d.sum()), len(filt))
