"""Per-CTA timeline of a stream-K / K-split launch (MYD_KS_TIMELINE build; development aid):

  python -m paper_1609_00076_b200.build -DMYD_KS_TIMELINE --out=build/variants/libkst.so
  MY_DGEMM_LIB=build/variants/libkst.so python tools/ksplit_timeline.py 1024 1024 1024 [strips]

Consumer warp 0 of every CTA: microseconds from the first CTA's entry to each mark."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import _capi, engine

lib = _capi.load()
fn = lib.my_dgemm_ks_timeline
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
m, n, k = (int(x) for x in sys.argv[1:4])
strips = int(sys.argv[4]) if len(sys.argv) > 4 else 48
st = torch.cuda.current_stream().cuda_stream
a = torch.rand(m * k, dtype=torch.float64, device="cuda")
b = torch.rand(k * n, dtype=torch.float64, device="cuda")
c = torch.rand(m * n, dtype=torch.float64, device="cuda")
run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=strips)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (160 * 16))()
fn(buf, 1)
run()
torch.cuda.synchronize()
fn(buf, 0)
rows = [list(buf[i * 16:(i + 1) * 16]) for i in range(160)]
rows = [r for r in rows if r[15]]
t0 = min(r[15] for r in rows)
us = lambda x: (x - t0) / 1e3 if x else float("nan")  # noqa: E731
names = ["s0 acc", "s0 loop", "s0 part/fix", "s0 stored", "s1 acc", "s1 start", "s1 loop", "s1 part/fix", "s1 stored",
         "s2 acc"]
print(f"{m}x{n}x{k} strips={strips}: {len(rows)} CTAs; last exit {max(us(r[14]) for r in rows):.2f} us")
print("cta  entry " + " ".join(f"{x:>11s}" for x in names) + "   exit")
for i, r in enumerate(rows):
    if i < 12 or i % 16 == 0 or i >= len(rows) - 4:
        print(f"{i:3d} {us(r[15]):6.2f} " + " ".join(f"{us(r[j]):11.2f}" for j in range(10)) + f" {us(r[14]):6.2f}")
import statistics
for j, nm in [(15, "entry"), (0, "s0 acc"), (1, "s0 loop"), (2, "s0 part/fix"), (3, "s0 stored"), (4, "s1 acc"),
              (6, "s1 loop"), (7, "s1 part/fix"), (8, "s1 stored"), (14, "exit")]:
    vals = [us(r[j]) for r in rows if r[j]]
    if vals:
        print(f"{nm:>12s}: n={len(vals):3d} mean {statistics.mean(vals):7.2f} max {max(vals):7.2f}")
