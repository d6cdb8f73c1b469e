"""Per-key cost of the four ops vs table size on one B200 (configs[3]'s
per-GPU shards: 2^24..2^27 buckets, f=16 b=16, 95 % load).

    python tools/table_scale.py [log2_buckets ...]   # default 24 25 26 27

One line per table: schedule + region runs per call, ms and ns/key per op
(CUDA events on the launching stream, second of two repetitions).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_15486_b200 import CuckooFilter, FilterConfig  # noqa: E402


def main() -> None:
    lms = [int(x) for x in sys.argv[1:]] or [24, 25, 26, 27]
    for lm in lms:
        cfg = FilterConfig(bucket_count=1 << lm, eviction="bfs", seed=0)
        n = int(0.95 * cfg.total_slots)
        g = torch.Generator(device="cuda").manual_seed(lm)
        pos = torch.randint(0, 1 << 62, (n,), device="cuda", generator=g, dtype=torch.int64)
        neg = torch.randint(1 << 62, (1 << 63) - 1, (n,), device="cuda", generator=g, dtype=torch.int64)
        filt = CuckooFilter(cfg)
        s = torch.cuda.current_stream()
        out = {}
        for rep in range(2):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            ev[0].record(s)
            r = filt.insert_batch(pos)
            sched = filt.last_schedule
            ev[1].record(s)
            filt.query_batch(pos)
            ev[2].record(s)
            filt.query_batch(neg)
            ev[3].record(s)
            filt.delete_batch(pos)
            ev[4].record(s)
            torch.cuda.synchronize()
            failed = r.n_failed
            del r
            ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
            out = {"log2_buckets": lm, "slots": cfg.total_slots, "keys": n, "schedule": sched,
                   "insert_failures": failed, "occupancy_after": len(filt)}
            for name, t in zip(("insert", "lookup+", "lookup-", "delete"), ms):
                out[name] = {"ms": round(t, 3), "ns_per_key": round(t * 1e6 / n, 4)}
            out["step_ns_per_key"] = round(sum(ms) * 1e6 / n, 4)
        print(json.dumps(out), flush=True)
        del filt, pos, neg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
