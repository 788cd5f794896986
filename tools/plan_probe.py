"""Device time per launch plan (heuristic, every tile as 128x64 / 128x32 /
64x32 units) over square sizes -- data for the plan cost model (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

sizes = [int(x) for x in sys.argv[1:]] or [768, 1024, 1280, 1536, 1792, 2048, 2304, 2560, 2816, 3072, 3328, 3584,
                                           3840]
st = torch.cuda.current_stream().cuda_stream
for s in sizes:
    a = torch.rand(s * s, dtype=torch.float64, device="cuda")
    b = torch.rand(s * s, dtype=torch.float64, device="cuda")
    c = torch.rand(s * s, dtype=torch.float64, device="cuda")
    inner = max(1, int(2e10 / (2.0 * s ** 3)))
    res = {}
    for strips in (0, 2, 4, 8, 32, 34, 36, 40):
        def go():
            for _ in range(inner):
                engine.dgemm_device(s, s, s, a.data_ptr(), s, b.data_ptr(), s, c.data_ptr(), s, st, strips=strips)
        go()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            go()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
        res[strips] = best
    plan, ms = engine.tune(s, s, s, reps=5)
    tiles = ((s + 127) // 128) ** 2
    print(f"{s}: tiles {tiles} ({tiles / 148:.2f} waves)  " +
          "  ".join(f"s{k}={v:.1f}us({2 * s ** 3 / v / 1e6 / 37.22 * 100:.0f}%)" for k, v in res.items()) +
          f"  tuned plan {plan} {ms * 1e3:.1f}us", flush=True)
    del a, b, c
