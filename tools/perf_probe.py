"""Quick device-resident timing probe of the fast kernel (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

def probe(m, n, k, reps=5, **kw):
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
    best = min(times)
    tf = 2.0 * m * n * k / best / 1e9
    print(f"{m}x{n}x{k} {kw}: best {best:.3f} ms  {tf:.2f} TFLOP/s  ({tf/37.22*100:.1f}% of 37.22)", flush=True)

quick = "--quick" in sys.argv
strips = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--strips=")] or [0]
sizes = [int(x) for x in sys.argv[1:] if not x.startswith("--")] or ([4096, 8192] if quick else [1024, 2048, 4096, 8192])
for s in sizes:
    for st_ in strips:
        probe(s, s, s, **({"strips": st_} if st_ else {}))
probe(16384, 16384, 256)
probe(4093, 4099, 2047)
if not quick:
    probe(8192, 8192, 8192, reps=2, exact=True)
