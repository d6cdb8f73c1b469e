"""f=32 (b=16, 64-byte buckets) at 2^28 slots: region vs direct schedule by batch size (G ops/s)."""
import sys
sys.path.insert(0, ".")
import json
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

OPS = ("insert", "lookup+", "lookup-", "delete")
for lb in (24, 26, 28):
    for tiled in (True, False):
        cfg = FilterConfig(bucket_count=1 << 24, fingerprint_bits=32, bucket_slots=16, eviction="bfs", seed=0)
        n = int(0.95 * cfg.total_slots)
        g = torch.Generator(device="cuda").manual_seed(5)
        pos = torch.randint(0, 1 << 62, (n,), device="cuda", generator=g, dtype=torch.int64)
        neg = torch.randint(1 << 62, (1 << 63) - 1, (n,), device="cuda", generator=g, dtype=torch.int64)
        filt = CuckooFilter(cfg, tiled=tiled)
        bs = min(n, 1 << lb)
        s = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        calls = (filt.insert_batch, filt.query_batch, filt.query_batch, filt.delete_batch)
        for j, (o, call) in enumerate(zip(OPS, calls)):
            src = neg if o == "lookup-" else pos
            ev[j].record(s)
            for lo in range(0, n, bs):
                call(src[lo: lo + bs])
            ev[j + 1].record(s)
        torch.cuda.synchronize()
        print(json.dumps({"f": 32, "batch": bs, "tiled": tiled, "schedule": filt.last_schedule,
                          "G_ops_s": {o: round(n / ev[j].elapsed_time(ev[j + 1]) / 1e6, 2) for j, o in enumerate(OPS)}}),
              flush=True)
        del filt, pos, neg
        torch.cuda.empty_cache()
