"""Planner regret scan (development aid): for seeded random shapes, the heuristic's time
against the best forced plan (full tiles, units, stream-K over tiles / units), back-to-back
calls.  Shapes where the heuristic loses more than 2 % are the planner's mis-picks.

    python tools/planner_regret.py [count] [seed]
"""
import os
import random
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

PLANS = {0: "heuristic", 1: "tiles", 2: "128x64", 4: "128x32", 8: "64x32", 32: "SK tiles", 34: "SK 128x64",
         36: "SK 128x32", 40: "SK 64x32", 64: "small"}
count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 7)


def dim(lo, hi, ragged):
    v = int(round(2 ** rng.uniform(lo, hi)))
    return v if ragged else max(128, v // 128 * 128)


shapes = []
for i in range(count):
    ragged = i % 3 == 2
    shapes.append((dim(8.5, 12.6, ragged), dim(8.5, 12.6, ragged), dim(6.5, 12.0, ragged) // 16 * 16 or 64))
st = torch.cuda.current_stream().cuda_stream
worst = []
for (m, n, k) in shapes:
    if 8.0 * (m * k + k * n + m * n) > 8e9:
        continue
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    res = {}
    for p, name in PLANS.items():
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)  # noqa: E731
        try:
            run(); run(); torch.cuda.synchronize()
        except Exception:
            continue
        inner = max(2, min(50, int(1.5e9 / (2.0 * m * n * k))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(inner):
                run()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
        res[name] = best
    h = res["heuristic"]
    bname = min(res, key=res.get)
    regret = h / res[bname] - 1.0
    frac = 2.0 * m * n * k / h / 1e6 / 37.22
    tiles = -(-m // 128) * -(-n // 128)
    print(f"{m}x{n}x{k} tiles={tiles} ({tiles / 148:.2f} waves): heuristic {h:.1f} us ({frac * 100:.1f} %), best {bname} "
          f"{res[bname]:.1f} us, regret {regret * 100:.1f} %" + ("  <<<" if regret > 0.02 else ""), flush=True)
    worst.append((regret, m, n, k, bname))
worst.sort(reverse=True)
print("mean regret %.2f %%, worst %s" % (100 * sum(w[0] for w in worst) / len(worst), worst[:5]))
