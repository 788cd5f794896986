"""Few-row shapes (2 <= m <= 32): the DMMA row kernel (PATH_ROWS_DMMA) vs the
FMA few-row kernel (PATH_FEW_ROWS, m <= 16) and the tiled kernel, device
time and GB/s over 8(mk + kn + 2mn); each checked against the exact kernel
(development aid).  Args: MxNxK shapes; MY_DGEMM_RD_CT=1|2|4 pins the
column-block width."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import _capi, engine

st = torch.cuda.current_stream().cuda_stream
EPS = 2.0 ** -53


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return best


shapes = [(2, 8192, 8192), (4, 8192, 8192), (8, 8192, 8192), (12, 8192, 8192), (16, 8192, 8192),
          (24, 8192, 8192), (32, 8192, 8192), (16, 4096, 4096), (8, 32768, 8192), (16, 65536, 2048),
          (8, 2048, 2048), (16, 1024, 8192), (5, 100000, 1000), (32, 16384, 4096)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for m, n, k in shapes:
    torch.manual_seed(0)
    a = torch.rand(m * k, dtype=torch.float64, device="cuda") * 2 - 1
    b = torch.rand(k * n, dtype=torch.float64, device="cuda") * 2 - 1
    c = torch.rand(m * n, dtype=torch.float64, device="cuda") * 2 - 1
    ce = c.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, ce.data_ptr(), m, st, exact=True)
    byts = 8.0 * (m * k + k * n + 2 * m * n)
    parts = []
    for name, p in (("rows_dmma", _capi.PATH_ROWS_DMMA), ("few_rows", _capi.PATH_FEW_ROWS), ("tiled", _capi.PATH_TILED)):
        if p == _capi.PATH_FEW_ROWS and m > 16:
            continue
        cc = c.clone()
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m, st, path=p)
        torch.cuda.synchronize()
        err = (cc - ce).abs().max().item() / (k * EPS * (k + 1))
        us = timed(lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m, st, path=p))
        parts.append(f"{name} {us:7.1f} us ({byts / us / 1e3:5.0f} GB/s, err/bound {err:.2e})")
    print(f"{m}x{n}x{k} [default path {engine.path(m, n)}]: " + " | ".join(parts), flush=True)
