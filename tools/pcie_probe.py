"""H2D / D2H pinned-copy throughput on the box (sizes like one bench op)."""
import time
import torch
n = 255 << 20
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
d = torch.empty(n, dtype=torch.int64, device="cuda")
o = torch.empty(n, dtype=torch.uint8, pin_memory=True)
do = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D {8*n/1e9:.2f} GB: {8*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
    torch.cuda.synchronize(); t = time.perf_counter(); o.copy_(do, non_blocking=True); torch.cuda.synchronize()
    print(f"D2H {n/1e9:.2f} GB: {n/(time.perf_counter()-t)/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): o.copy_(do, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"concurrent H2D {8*n/1e9:.2f} GB + D2H {n/1e9:.2f} GB: {dt*1e3:.1f} ms")
