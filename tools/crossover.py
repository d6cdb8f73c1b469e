"""Direct vs region schedule by batch size (the automatic choice's crossover).

    python tools/crossover.py  -> one JSON line per (f, batch, schedule)

A 2^28-slot b=16 table (f=16: 512 MiB, f=32: 1 GiB) filled to 95 % in batches
of the given size, then lookup+ / lookup- / delete in the same batches; the
second of two repetitions (the first grows the workspace)."""
import sys
sys.path.insert(0, ".")
import json
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

OPS = ("insert", "lookup+", "lookup-", "delete")
for f in (16, 32):
    for lb in (22, 23, 24, 25, 26):
        for tiled in (True, False):
            cfg = FilterConfig(bucket_count=1 << 24, fingerprint_bits=f, bucket_slots=16, eviction="bfs", seed=0)
            n = int(0.95 * cfg.total_slots)
            g = torch.Generator(device="cuda").manual_seed(5)
            pos = torch.randint(0, 1 << 62, (n,), device="cuda", generator=g, dtype=torch.int64)
            neg = torch.randint(1 << 62, (1 << 63) - 1, (n,), device="cuda", generator=g, dtype=torch.int64)
            filt = CuckooFilter(cfg, tiled=tiled)
            bs = 1 << lb
            s = torch.cuda.current_stream()
            for rep in range(2):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                calls = (filt.insert_batch, filt.query_batch, filt.query_batch, filt.delete_batch)
                for j, (o, call) in enumerate(zip(OPS, calls)):
                    src = neg if o == "lookup-" else pos
                    ev[j].record(s)
                    for lo in range(0, n, bs):
                        call(src[lo: lo + bs])
                    ev[j + 1].record(s)
                torch.cuda.synchronize()
            ms = [ev[j].elapsed_time(ev[j + 1]) for j in range(4)]
            print(json.dumps({"f": f, "batch": bs, "n_over_m": round(bs / cfg.bucket_count, 3),
                              "schedule": "region" if tiled else "direct",
                              "G_ops_s": {o: round(n / t / 1e6, 2) for o, t in zip(OPS, ms)},
                              "total_ms": round(sum(ms), 2)}), flush=True)
            del filt, pos, neg
            torch.cuda.empty_cache()
