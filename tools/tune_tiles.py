"""Tile-parameter grid search per shape class (paper_1609_00076_b200.tuning.tune_grid,
the reference's tune() at several probe shapes): every compiled (bm, bn, bk,
stages) point timed and verified, the winner per class against the
heuristic's own plan (profiles/r02/tune_tiles_r02*.log).

  python tools/tune_tiles.py [MxNxK ...]
"""
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import _capi, engine, tuning

CLASSES = [(256, 256, 256), (512, 512, 512), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096),
           (4096, 4096, 256), (8192, 8192, 128), (128, 128, 4096), (1000, 1000, 64), (4093, 4099, 2047)]
if len(sys.argv) > 1:
    CLASSES = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
lib = _capi.load()
for m, n, k in CLASSES:
    lib.my_dgemm_tune_clear()
    log = io.StringIO()
    res = tuning.tune_grid({}, probe_size=max(m, n, k), reps=3, log=log, apply=False, shape=(m, n, k))
    # the heuristic's own time, same protocol
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 7 + t, 0, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    heur = float("inf")
    for _ in range(4):
        e0.record()
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
        e1.record()
        torch.cuda.synchronize()
        heur = min(heur, e0.elapsed_time(e1) * 1e-3)
    hr = 2.0 * m * n * k / heur / 1e9
    top = sorted(res.table.items(), key=lambda kv: -kv[1])[:4]
    b_ = res.best
    print(f"{m}x{n}x{k}: best bm={b_.bm} bn={b_.bn} bk={b_.bk} stages={b_.stages} (plan {b_.plan}) "
          f"{res.rate:.0f} GF/s ({res.rate / 37220 * 100:.1f} %) | heuristic {hr:.0f} GF/s | "
          f"points {len(res.table)} timed, {len(res.skipped)} skipped | next: "
          + ", ".join(f"{p.bm}x{p.bn}/{p.bk}/{p.stages} p{p.plan} {r:.0f}" for p, r in top[1:]), flush=True)
    del a, b, c
