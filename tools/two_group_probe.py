"""Two consumer groups per CTA (plan 3 -- an experiment removed after this
probe, see git history: 128x64 units, each group its own ring and unit
sequence, the second half a unit behind) against the heuristic, full tiles
and one-group 128x64 units: device time of back-to-back calls and a bitwise
check against the heuristic's C (profiles/r02/two_group_r02a.log).

  python tools/two_group_probe.py [MxNxK ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

PLANS = {0: "heur", 1: "tiles", 2: "128x64", 3: "2grp"}
if os.environ.get("PLANS"):
    PLANS = {int(p): n for p, n in (x.split(":") for x in os.environ["PLANS"].split(","))}
shapes = [(16384, 16384, 256), (16384, 16384, 128), (8192, 8192, 512), (12000, 12000, 100), (4096, 4096, 4096),
          (8192, 8192, 8192), (4093, 4099, 2047), (2048, 2048, 2048), (8192, 8192, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
st = torch.cuda.current_stream().cuda_stream
for (m, n, k) in shapes:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c0, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    ref = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, ref.data_ptr(), m, st)
    row = []
    for p, name in PLANS.items():
        cc = c0.clone()
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m, st, strips=p)
        torch.cuda.synchronize()
        same = torch.equal(cc, ref)
        del cc
        c = c0.clone()
        inner = max(1, int(2e11 / (2.0 * m * n * k)))
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st,  # noqa: E731
                                          strips=p)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record()
            for _ in range(inner):
                run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / inner)
        best = min(ts)
        tf = 2.0 * m * n * k / best / 1e6
        row.append(f"{name}: {best:.1f} us {tf / 37.22 * 100:.2f}%{'' if same else ' MISMATCH'}")
        del c
    print(f"{m}x{n}x{k} | " + " | ".join(row), flush=True)
    del a, b, c0, ref
    torch.cuda.empty_cache()
