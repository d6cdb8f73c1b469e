"""Time the routing partition vs torch's stable argsort at 2^28 keys, 8 shards."""
import sys
import time
sys.path.insert(0, ".")
import torch
from paper_2603_15486_b200 import _lib


def route(h, shift, shards):
    L = _lib.lib()
    n = h.numel()
    send = torch.empty_like(h)
    order = torch.empty(n, dtype=torch.int64, device=h.device)
    counts = torch.empty(shards, dtype=torch.int64, device=h.device)
    wsb = int(L.ckf_route_workspace_bytes(n, shards))
    ws = torch.empty(wsb, dtype=torch.uint8, device=h.device)
    _lib.check(L.ckf_route_partition(h.data_ptr(), n, shift, shards, send.data_ptr(), order.data_ptr(),
                                     counts.data_ptr(), ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream))


n = 255_013_683
h = torch.randint(0, 1 << 62, (n,), device="cuda", dtype=torch.int64)
for name, fn in [("ckf_route_partition", lambda: route(h, 61, 8)),
                 ("torch stable argsort(uint8) + gather", lambda: h[torch.argsort(torch.bitwise_and(h >> 61, 7).to(torch.uint8), stable=True)])]:
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{name}: {dt * 1e3:.2f} ms for {n} hashes")
