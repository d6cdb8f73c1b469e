"""BASELINE configs[4] throughput: mixed 50/25/25 lookup/insert/delete stream.

2^28 slots, b=16, f in {8, 16, 32}, prefilled to 50 %.  Each round issues one
batch of B/4 inserts of new keys, one batch of B/4 deletes of keys inserted in
earlier rounds and one batch of B/2 lookups of keys whose membership is fixed
within the round (the correctness side is
tests/test_gpu_configs.py::test_mixed_stream_fpr).  Device time of all rounds
(CUDA events), keys resident in HBM; B = 2^26 ops per round.  Two forms:
"phases" (three batch calls per round: insert, delete, lookup) and "fused"
(CuckooFilter.mixed_batch: the round's shuffled ops in ONE concurrent launch).

    python tools/mixed_stream.py  -> profiles/r02_mixed_stream.txt
"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

B = 1 << 26
ROUNDS = 6
lines = []
for mode, f in [(m, f) for f in (8, 16, 32) for m in ("phases", "fused")]:
    cfg = FilterConfig(bucket_count=(1 << 28) // 16, fingerprint_bits=f, bucket_slots=16, eviction="bfs")
    slots = cfg.total_slots
    g = torch.Generator(device="cuda")
    g.manual_seed(f)
    pool = torch.randint(0, 1 << 62, (slots // 2 + (ROUNDS + 1) * B // 4,), device="cuda", dtype=torch.int64,
                         generator=g)
    filt = CuckooFilter(cfg)
    filt.insert_batch(pool[: slots // 2])
    head, nxt = 0, slots // 2  # live keys = pool[head:nxt] (deletes take the oldest)
    rounds = []  # (new, doomed, probe) per round, built before timing
    for r in range(ROUNDS + 1):
        new = pool[nxt + r * B // 4: nxt + (r + 1) * B // 4]
        doomed = pool[head + r * B // 4: head + (r + 1) * B // 4]
        idx = torch.randint(head + (r + 1) * B // 4, nxt + r * B // 4, (B // 2,), device="cuda", generator=g)
        probe = pool[idx]
        if mode == "fused":
            keys = torch.cat([new, doomed, probe])
            ops = torch.cat([torch.full((B // 4,), 1, dtype=torch.uint8, device="cuda"),
                             torch.full((B // 4,), 2, dtype=torch.uint8, device="cuda"),
                             torch.zeros(B // 2, dtype=torch.uint8, device="cuda")])
            perm = torch.randperm(B, device="cuda", generator=g)
            rounds.append((ops[perm].contiguous(), keys[perm].contiguous()))
        else:
            rounds.append((new, doomed, probe))
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    for r in range(ROUNDS + 1):  # round 0 is an untimed warm-up
        if r == 1:
            torch.cuda.synchronize()
            s.record()
        if mode == "phases":
            new, doomed, probe = rounds[r]
            filt.insert_batch(new)
            filt.delete_batch(doomed)
            hits = filt.query_batch(probe)
        else:
            ops, keys = rounds[r]
            hits = filt.mixed_batch(ops, keys)
    head += (ROUNDS + 1) * B // 4
    nxt += (ROUNDS + 1) * B // 4
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    ok = bool(hits.all()) and len(filt) == nxt - head
    line = (f"{mode} f={f}: {ROUNDS} rounds x {B} ops (50% lookup / 25% insert / 25% delete) at ~50% load: "
            f"{ROUNDS * B / ms / 1e6:.1f} G ops/s ({ms / ROUNDS:.2f} ms/round); no false negatives & occupancy ok: {ok}")
    print(line, flush=True)
    lines.append(line)
open("profiles/r02_mixed_stream.txt", "w").write("\n".join(lines) + "\n")
