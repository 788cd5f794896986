"""Is a unit shape bound by aggregate L2 bandwidth or by the SM itself?
Per-SM throughput of every-tile-as-units plans at 148 / 74 / 37 persistent
CTAs (my_dgemm_set_max_ctas): if the narrow units run faster per SM when
fewer SMs share the L2, the aggregate L2 -> SM bandwidth is the limit
(development aid; profiles/l2_bound_probe_r01.log)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
a = torch.empty(m * k, dtype=torch.float64, device="cuda")
b = torch.empty(k * n, dtype=torch.float64, device="cuda")
c = torch.empty(m * n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
    engine.fill_random_device(buf.data_ptr(), r, cc, r, 7 + t, 0, st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for strips, name in ((1, "128x128"), (2, "128x64"), (4, "128x32"), (8, "64x32"), (16, "16x128")):
    for ctas in (148, 74, 37):
        prev = engine.set_max_ctas(ctas)
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=strips)
        run(); run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        engine.set_max_ctas(prev)
        t = min(ts) * 1e-3
        per_sm = 2.0 * m * n * k / t / ctas / 1e9
        print(f"{m}^3 units {name:8s} ctas {ctas:3d}: {t*1e6:9.1f} us  {per_sm:6.1f} GFLOP/s per SM "
              f"({per_sm / 251.5 * 100:5.1f}% of the SM's DMMA rate)", flush=True)
