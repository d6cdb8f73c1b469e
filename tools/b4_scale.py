"""b=4 (one 8-byte word per bucket, f=16) at 2^28 slots: region vs direct (G ops/s)."""
import sys
sys.path.insert(0, ".")
import json
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

OPS = ("insert", "lookup+", "lookup-", "delete")
for tiled in (None, False):
    cfg = FilterConfig(bucket_count=1 << 26, fingerprint_bits=16, bucket_slots=4, eviction="bfs", seed=0)
    n = int(0.95 * cfg.total_slots)
    g = torch.Generator(device="cuda").manual_seed(3)
    pos = torch.randint(0, 1 << 62, (n,), device="cuda", generator=g, dtype=torch.int64)
    neg = torch.randint(1 << 62, (1 << 63) - 1, (n,), device="cuda", generator=g, dtype=torch.int64)
    filt = CuckooFilter(cfg, tiled=tiled)
    best = {o: 1e9 for o in OPS}
    for _ in range(2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(); r = filt.insert_batch(pos); sch = filt.last_schedule; ev[1].record()
        filt.query_batch(pos); ev[2].record(); filt.query_batch(neg); ev[3].record()
        filt.delete_batch(pos[r.ok]); ev[4].record(); torch.cuda.synchronize()
        for j, o in enumerate(OPS):
            best[o] = min(best[o], ev[j].elapsed_time(ev[j + 1]))
        failed = r.n_failed
        filt.clear()
    print(json.dumps({"b": 4, "slots": cfg.total_slots, "schedule": sch, "insert_failures": failed,
                      "G_ops_s": {o: round(n / best[o] / 1e6, 2) for o in OPS}}), flush=True)
