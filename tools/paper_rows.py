"""The paper's comparison rows on one B200 (PAPER.md:688-712 bucket-policy
figure: XOR vs Offset, L2- vs DRAM-resident, 95 % load; and the batch-size
dependence of the DRAM-resident numbers).

    python tools/paper_rows.py  -> profiles/r02_paper_rows.jsonl

Rows (G ops/s per op, CUDA events around each op's call, keys resident):
  * policy x residency: {xor, offset} x {2^22 slots (8 MiB table, L2-resident),
    2^28 slots (512 MiB, DRAM-resident)}; offset uses prime bucket counts
    (262 139 and 16 777 213), the case the policy exists for;
  * batch size: 2^28 slots, the same 0.95 * 2^28 keys issued in batches of
    2^20 .. 2^28 keys (the schedule each batch size gets is reported).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_15486_b200 import CuckooFilter, FilterConfig  # noqa: E402

OPS = ("insert", "lookup+", "lookup-", "delete")


def run(cfg: FilterConfig, batch: int | None = None, reps: int = 3) -> dict:
    n = int(0.95 * cfg.total_slots)
    g = torch.Generator(device="cuda").manual_seed(7)
    pos = torch.randint(0, 1 << 62, (n,), device="cuda", generator=g, dtype=torch.int64)
    neg = torch.randint(1 << 62, (1 << 63) - 1, (n,), device="cuda", generator=g, dtype=torch.int64)
    filt = CuckooFilter(cfg)
    bs = batch or n
    s = torch.cuda.current_stream()
    best = {o: float("inf") for o in OPS}
    sched = {}
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        calls = (lambda k: filt.insert_batch(k), filt.query_batch, filt.query_batch, filt.delete_batch)
        for j, (o, call) in enumerate(zip(OPS, calls)):
            src = neg if o == "lookup-" else pos
            ev[j].record(s)
            for lo in range(0, n, bs):
                call(src[lo: lo + bs])
            sched[o] = filt.last_schedule
            ev[j + 1].record(s)
        torch.cuda.synchronize()
        for j, o in enumerate(OPS):
            best[o] = min(best[o], ev[j].elapsed_time(ev[j + 1]))
    assert len(filt) == 0
    return {"slots": cfg.total_slots, "buckets": cfg.bucket_count, "policy": cfg.policy.value, "keys": n,
            "batch": bs, "schedule": {o: list(v) for o, v in sched.items()},
            "G_ops_s": {o: round(n / best[o] / 1e6, 2) for o in OPS},
            "ms": {o: round(best[o], 3) for o in OPS}}


def main() -> None:
    rows = []
    for log2, m_off in ((22, 262_139), (28, 16_777_213)):
        for pol, m in (("xor", 1 << (log2 - 4)), ("offset", m_off)):
            r = run(FilterConfig(bucket_count=m, policy=pol, eviction="bfs", seed=0))
            r["row"] = f"policy {pol}, {'L2' if log2 == 22 else 'DRAM'}-resident"
            rows.append(r)
            print(json.dumps(r), flush=True)
    for lb in (20, 22, 24, 26, 28):
        r = run(FilterConfig(bucket_count=1 << 24, eviction="bfs", seed=0), batch=1 << lb, reps=2)
        r["row"] = f"batch 2^{lb} keys"
        rows.append(r)
        print(json.dumps(r), flush=True)
    Path("profiles/r02_paper_rows.jsonl").write_text("\n".join(json.dumps(r) for r in rows) + "\n")


if __name__ == "__main__":
    main()
