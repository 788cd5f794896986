"""A/B: stream-K over every tile (MY_DGEMM_SK_DP_WAVES=w) vs the default plan (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine


def probe(m, n, k, reps=7, **kw):
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (r, cc) in enumerate(((m, k), (k, n), (m, n))):
        engine.fill_random_device([a, b, c][t].data_ptr(), r, cc, r, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, **kw)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(reps):
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    tf = 2.0 * m * n * k / times[0] / 1e9
    print(f"{m}x{n}x{k} {kw} waves={os.environ.get('MY_DGEMM_SK_DP_WAVES')}: best {times[0]*1e3:.1f} us "
          f"median {times[len(times)//2]*1e3:.1f} us  {tf:.2f} TF ({tf/37.22*100:.1f}%)", flush=True)


shapes = [(16384, 16384, 256), (16384, 16384, 128), (16384, 16384, 512), (8192, 8192, 256), (2048, 2048, 2048),
          (4096, 4096, 4096), (8192, 8192, 8192), (4093, 4099, 2047)]
for s in shapes:
    for strips in (0, 32):
        probe(*s, **({"strips": strips} if strips else {}))
