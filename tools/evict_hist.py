"""Histogram of eviction rounds of the bench insert (2^28 slots, 95 % load)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

cfg = FilterConfig(bucket_count=1 << 24, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda").manual_seed(0)
pos = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64, generator=g)
filt = CuckooFilter(cfg)
r = filt.insert_batch(pos)
rec = r.records()
ev = rec["evictions"]
h = np.bincount(ev.astype(np.int64))
print("queued", len(rec), "failed", int((rec["ok"] == 0).sum()))
print("rounds histogram", {i: int(c) for i, c in enumerate(h) if c})
w = ev[: len(ev) // 32 * 32].reshape(-1, 32)
print("mean rounds", ev.mean(), "mean warp max (32 consecutive queue entries)", w.max(1).mean())
