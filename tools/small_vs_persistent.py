"""Small-block kernel vs the persistent kernel's plans on seeded random shapes of up to two waves
of tiles (where the planner compares the two cost models): measured time of the small kernel's
model pick (plan 64) and of the best forced persistent plan, against the two models' predictions
(tuning.describe_plan: small_us, model_us).  Calibration evidence for the crossover
(profiles/r02/small_vs_persistent_r02a.log).

    python tools/small_vs_persistent.py [count] [seed]
"""
import os
import random
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine, tuning

PERS = (1, 2, 4, 8, 32, 34, 36, 40)
count = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
st = torch.cuda.current_stream().cuda_stream


def timed(m, n, k, a, b, c, p):
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)  # noqa: E731
    try:
        run(); run(); torch.cuda.synchronize()
    except Exception:
        return None
    inner = max(3, min(100, int(1e9 / (2.0 * m * n * k))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(inner):
            run()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
    return best


rows = []
while len(rows) < count:
    ragged = len(rows) % 3 == 2
    m = int(round(2 ** rng.uniform(7.0, 12.3)))
    n = int(round(2 ** rng.uniform(7.0, 12.3)))
    k = max(32, int(round(2 ** rng.uniform(5.5, 12.0))) // 16 * 16)
    if not ragged:
        m, n = max(128, m // 64 * 64), max(128, n // 64 * 64)
    tiles = -(-m // 128) * -(-n // 128)
    if tiles > 296 or m * n * k < 2e6:
        continue
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    d = tuning.describe_plan(m, n, k)
    ts = timed(m, n, k, a, b, c, 64)
    tp = min(x for x in (timed(m, n, k, a, b, c, p) for p in PERS) if x is not None)
    th = timed(m, n, k, a, b, c, 0)
    rows.append((m, n, k, tiles, d["kind"], d["model_us"], d["small_us"], tp, ts, th))
    print(f"{m}x{n}x{k} tiles={tiles} pick={d['kind']}: persistent model {d['model_us']:.1f} meas {tp:.1f} "
          f"(x{tp / d['model_us']:.2f}) | small model {d['small_us']:.1f} meas {ts:.1f} (x{ts / d['small_us']:.2f}) | "
          f"heuristic {th:.1f} vs best {min(tp, ts):.1f} ({(th / min(tp, ts) - 1) * 100:+.1f} %)", flush=True)
import statistics
rp = [r[7] / r[5] for r in rows]
rs = [r[8] / r[6] for r in rows]
print(f"measured / model: persistent median {statistics.median(rp):.3f} mean {statistics.mean(rp):.3f}; "
      f"small median {statistics.median(rs):.3f} mean {statistics.mean(rs):.3f}")
for f in (0.85, 0.9, 0.95, 1.0, 1.05, 1.1):
    tot = sum((r[8] if r[6] * f < r[5] else r[7]) / min(r[7], r[8]) for r in rows) / len(rows)
    print(f"small model x{f}: mean time over best {100 * (tot - 1):.2f} %")
