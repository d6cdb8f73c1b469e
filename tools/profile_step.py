"""One warm-up + one profiled step of the bench protocol (for ncu launch lists).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py [--tiled auto|on|off]
"""
import argparse
import sys
sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2603_15486_b200 import CuckooFilter, FilterConfig

ap = argparse.ArgumentParser()
ap.add_argument("--log2-slots", type=int, default=28)
ap.add_argument("--tiled", default="auto", choices=["auto", "on", "off"])
ap.add_argument("--eviction", default="bfs")
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()
tiled = {"auto": None, "on": True, "off": False}[args.tiled]
cfg = FilterConfig(bucket_count=(1 << args.log2_slots) // 16, eviction=args.eviction)
n = int(0.95 * cfg.total_slots)
g = torch.Generator(device="cuda")
g.manual_seed(0)
pos = torch.randint(0, 1 << 32, (n,), device="cuda", dtype=torch.int64, generator=g)
neg = torch.randint(1 << 32, 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)
filt = CuckooFilter(cfg, tiled=tiled)
for _ in range(args.steps):
    r = filt.insert_batch(pos)
    c = r._ctr.cpu().tolist()
    print("insert counters n_ok=%d records=%d queued=%d alt=%d" % tuple(c))
    filt.query_batch(pos)
    print("lookup+", filt.last_counters())
    filt.query_batch(neg)
    filt.delete_batch(pos)
    print("delete", filt.last_counters())
torch.cuda.synchronize()
print("occupancy", len(filt))
