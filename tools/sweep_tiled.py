"""Time the four ops (direct vs tiled, tiled knobs) on the bench config.

    python tools/sweep_tiled.py            # prints one line per setting
Settings are passed through CKF_REGION_KB / CKF_BIN_GROUP (read per call).
"""
import itertools
import os
import sys

sys.path.insert(0, ".")
import torch

from paper_2603_15486_b200 import CuckooFilter, FilterConfig

log2 = int(os.environ.get("LOG2", 28))
cfg = FilterConfig(bucket_count=(1 << log2) // 16, eviction="bfs")
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda")
g.manual_seed(0)
pos = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64, generator=g)
neg = torch.randint(1 << 32, 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)


def run(tiled, reps=3):
    filt = CuckooFilter(cfg, tiled=tiled)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    best = [1e9] * 4
    for _ in range(reps):
        ev[0].record()
        r = filt.insert_batch(pos)
        ev[1].record()
        filt.query_batch(pos)
        ev[2].record()
        q = filt.query_batch(neg)
        ev[3].record()
        d = filt.delete_batch(pos)
        ev[4].record()
        torch.cuda.synchronize()
        best = [min(b, ev[i].elapsed_time(ev[i + 1])) for i, b in enumerate(best)]
    ok = r.n_failed == 0 and bool(d.all()) and len(filt) == 0
    fpr = float(q.float().mean())
    del filt
    torch.cuda.empty_cache()
    return best, ok, fpr


def show(tag, best, ok, fpr):
    tot = sum(best)
    print(f"{tag:<28} ins {best[0]:6.2f}  q+ {best[1]:6.2f}  q- {best[2]:6.2f}  del {best[3]:6.2f}  "
          f"step {tot:6.2f} ms  {4 * n / tot / 1e6:6.2f} Gops/s  ok={ok} fpr={fpr:.2e}", flush=True)


show("direct", *run(False))
regions = [int(x) for x in os.environ.get("REGIONS", "1024,2048").split(",")]
groups = [int(x) for x in os.environ.get("BINGROUPS", "4,8,32").split(",")]
for reg, grp in itertools.product(regions, groups):
    os.environ["CKF_REGION_KB"] = str(reg)
    os.environ["CKF_BIN_GROUP"] = str(grp)
    show(f"tiled region={reg}KB group={grp}", *run(True))
