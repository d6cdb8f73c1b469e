"""Quick device-side throughput probe of the direct kernels (dev tool, not the bench)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2603_15486_b200 import CuckooFilter, FilterConfig

def timeit(fn, reps=3):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best

for logslots, b, ev in [(22, 16, 'bfs'), (28, 16, 'bfs'), (28, 16, 'dfs'), (20, 4, 'bfs')]:
    m = (1 << logslots) // b
    cfg = FilterConfig(bucket_count=m, bucket_slots=b, eviction=ev)
    n = int(0.95 * cfg.total_slots)
    g = torch.Generator(device='cuda'); g.manual_seed(0)
    keys = torch.randint(0, 1 << 32, (n,), device='cuda', dtype=torch.int64, generator=g)
    neg = torch.randint(1 << 32, 1 << 62, (n,), device='cuda', dtype=torch.int64, generator=g)
    filt = CuckooFilter(cfg)
    def ins():
        filt.clear(); filt.insert_batch(keys)
    t_ins = timeit(ins)
    r = filt.insert_batch.__self__  # noqa
    filt.clear(); res = filt.insert_batch(keys); nf = res.n_failed
    t_qp = timeit(lambda: filt.query_batch(keys))
    t_qn = timeit(lambda: filt.query_batch(neg))
    fpr = float(filt.query_batch(neg).float().mean())
    def dl():
        filt.delete_batch(keys)
    # delete needs a full table each rep
    best = 1e9
    for _ in range(3):
        filt.clear(); filt.insert_batch(keys); torch.cuda.synchronize()
        best = min(best, timeit(dl, 1))
    t_del = best
    clr = timeit(lambda: filt.clear())
    print(f"2^{logslots} b={b} {ev}: n={n} failed={nf} fpr={fpr:.3e} | insert {n/(t_ins-clr)/1e6:.2f} G/s  "
          f"lookup+ {n/t_qp/1e6:.2f}  lookup- {n/t_qn/1e6:.2f}  delete {n/t_del/1e6:.2f} G/s  (ms: {t_ins:.2f} {t_qp:.2f} {t_qn:.2f} {t_del:.2f})", flush=True)
