"""Per-plan timing of mid-size problems, back-to-back calls (PDL overlap), as
tools/sweep.py times them (development aid): which plan wins below ~1.5 waves."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

PLANS = {0: "heuristic", 2: "128x64", 4: "128x32", 8: "64x32", 32: "SK tiles", 34: "SK 128x64",
         36: "SK 128x32", 40: "SK 64x32"}
sizes = [int(x) for x in sys.argv[1:]] or [768, 1024, 1280, 1536, 1792]
for s in sizes:
    m = n = k = s
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    row = []
    for p, name in list(PLANS.items()) + [(0, "heuristic again")]:
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)
        try:
            for _ in range(3):
                run()
            torch.cuda.synchronize()
        except Exception as e:  # plan not applicable
            row.append(f"{name}: n/a")
            continue
        reps = max(5, int(2e6 / (s ** 3 / 1e3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
        tf = 2.0 * s ** 3 / best / 1e6
        row.append(f"{name}: {best:.1f} us {tf / 37.22 * 100:.1f}%")
    print(f"{s}^3 | " + " | ".join(row), flush=True)
    if os.environ.get("MIDSIZE_JSON"):
        with open(os.environ["MIDSIZE_JSON"], "a") as f:
            f.write(json.dumps({"size": s, "plans": {r.split(":")[0]: (float(r.split()[-3]) if "n/a" not in r else None)
                                                     for r in row}}) + "\n")
