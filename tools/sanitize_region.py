"""Small forced-region runs of insert / query / delete (compute-sanitizer target).

Covers the round-2 region pipeline: 8-byte records (f = 8 / 16, b = 16 / 32),
16-byte records (f = 32), one-word buckets (b = 4 at f = 16, odd-m offset
table: the plain-copied tail word), calls split into several region runs
(CKF_MAX_RUN_KEYS, set by the caller), the deferred-CAS retry ring and the
room map + BFS eviction (95 % load), and the one-launch mixed batch.
"""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

CASES = [(16, 16, "xor", 11), (8, 16, "offset", 11), (16, 32, "xor", 11), (32, 16, "xor", 11),
         (16, 4, "xor", 13), (16, 4, "offset", 13)]
for f, b, pol, lm in CASES:
    m = (1 << lm) - (3 if pol == "offset" else 0)
    cfg = FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b, policy=pol, eviction="bfs", seed=1)
    rng = np.random.default_rng(0)
    keys = rng.integers(0, 1 << 62, size=int(0.95 * cfg.total_slots), dtype=np.uint64)
    neg = rng.integers(1 << 62, 1 << 63, size=len(keys), dtype=np.uint64)
    filt = CuckooFilter(cfg, tiled=True)
    r = filt.insert_batch(keys)
    assert filt.last_schedule[0] == "region", filt.last_schedule
    q = filt.query_batch(keys)
    qn = filt.query_batch(neg)
    d = filt.delete_batch(keys)
    torch.cuda.synchronize()
    print(f, b, pol, filt.last_schedule, r.n_failed, bool(q.all()), float(qn.mean()), int(d.sum()), len(filt),
          flush=True)
    ops = rng.integers(0, 3, size=len(keys), dtype=np.uint8)
    filt.mixed_batch(ops, keys)
    torch.cuda.synchronize()
print("runs per call capped at", os.environ.get("CKF_MAX_RUN_KEYS", "default"))
