"""BASELINE configs[4] throughput: mixed 50/25/25 lookup/insert/delete stream.

2^28 slots, b=16, f in {8, 16, 32}, prefilled to 50 %.  Each round issues one
batch of B/4 inserts of new keys, one batch of B/4 deletes of keys inserted in
earlier rounds and one batch of B/2 lookups of keys whose membership is fixed
within the round (the correctness side is
tests/test_gpu_configs.py::test_mixed_stream_fpr).  Device time of all rounds
(CUDA events), keys resident in HBM; B = 2^26 ops per round.

    python tools/mixed_stream.py  -> profiles/r01s2_mixed_stream.txt
"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

B = 1 << 26
ROUNDS = 6
lines = []
for f in (8, 16, 32):
    cfg = FilterConfig(bucket_count=(1 << 28) // 16, fingerprint_bits=f, bucket_slots=16, eviction="bfs")
    slots = cfg.total_slots
    g = torch.Generator(device="cuda")
    g.manual_seed(f)
    pool = torch.randint(0, 1 << 62, (slots // 2 + (ROUNDS + 1) * B // 4,), device="cuda", dtype=torch.int64,
                         generator=g)
    filt = CuckooFilter(cfg)
    filt.insert_batch(pool[: slots // 2])
    head, nxt = 0, slots // 2  # live keys = pool[head:nxt] (deletes take the oldest)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    for r in range(ROUNDS + 1):  # round 0 is an untimed warm-up
        if r == 1:
            torch.cuda.synchronize()
            s.record()
        new = pool[nxt: nxt + B // 4]
        doomed = pool[head: head + B // 4]
        idx = torch.randint(head + B // 4, nxt, (B // 2,), device="cuda", generator=g)
        probe = pool[idx]
        filt.insert_batch(new)
        filt.delete_batch(doomed)
        hits = filt.query_batch(probe)
        head += B // 4
        nxt += B // 4
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    ok = bool(hits.all()) and len(filt) == nxt - head
    line = (f"f={f}: {ROUNDS} rounds x {B} ops (50% lookup / 25% insert / 25% delete) at ~50% load: "
            f"{ROUNDS * B / ms / 1e6:.1f} G ops/s ({ms / ROUNDS:.2f} ms/round); no false negatives & occupancy ok: {ok}")
    print(line, flush=True)
    lines.append(line)
open("profiles/r01s2_mixed_stream.txt", "w").write("\n".join(lines) + "\n")
