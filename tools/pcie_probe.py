"""Host<->device copy bandwidth with pinned and pageable buffers (e2e budget)."""
import time, torch, numpy as np
n = 512 * 1024 * 1024 // 8
d = torch.empty(n, dtype=torch.float64, device="cuda")
hp = torch.empty(n, dtype=torch.float64, pin_memory=True)
hn = torch.empty(n, dtype=torch.float64)
def bw(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9
print(f"H2D pinned   {bw(lambda: d.copy_(hp, non_blocking=True), n*8):.1f} GB/s")
print(f"D2H pinned   {bw(lambda: hp.copy_(d, non_blocking=True), n*8):.1f} GB/s")
print(f"H2D pageable {bw(lambda: d.copy_(hn), n*8, 3):.1f} GB/s")
print(f"D2H pageable {bw(lambda: hn.copy_(d), n*8, 3):.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d); hp2 = torch.empty_like(hp)
def duplex():
    with torch.cuda.stream(s1): d.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2): hp2.copy_(d2, non_blocking=True)
print(f"duplex H2D+D2H total {bw(duplex, 2*n*8):.1f} GB/s")
import os
print("host cpus", len(os.sched_getaffinity(0)))
