"""Kernel-internal timeline of a MYD_TIMELINE build (development aid):

  python -m paper_1609_00076_b200.build -DMYD_TIMELINE --out=build/variants/libtl.so
  MY_DGEMM_LIB=build/variants/libtl.so python tools/timeline_probe.py 512 512 16

globaltimer marks (ns, relative to the first CTA's entry) of CTA 0 / consumer
warp 0 for its first unit, the last CTA exit, and the graph-replayed device
time per call for comparison."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import _capi, engine

lib = _capi.load()
fn = lib.my_dgemm_timeline
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 32)()
shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]] or [(512, 512, 16), (512, 512, 512),
                                                                         (1024, 1024, 1024)]
for m, n, k in shapes:
    st = torch.cuda.current_stream().cuda_stream
    a = torch.rand(m * k, dtype=torch.float64, device="cuda")
    b = torch.rand(k * n, dtype=torch.float64, device="cuda")
    c = torch.rand(m * n, dtype=torch.float64, device="cuda")
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    marks = []
    for _ in range(5):
        fn(buf, 1)
        run()
        torch.cuda.synchronize()
        fn(buf, 0)
        v = list(buf)
        marks.append([(x - v[0]) / 1e3 if x else float("nan") for x in v])
    best = min(marks, key=lambda r: r[1])
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g, stream=s2):
            for _ in range(20):
                engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, s2.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) * 1e3 / 200
    print(f"{m}x{n}x{k}: graph {per:.2f} us/call; CTA span {best[1]:.2f} us; CTA0: init {best[2]:.2f}, "
          f"C ready {best[3]:.2f}, slab0 {best[4]:.2f}, loop end {best[5]:.2f}, epilogue {best[6]:.2f} us; "
          f"producer: start {best[8]:.2f}, unit0 {best[9]:.2f}, C slots issued {best[10]:.2f} {best[11]:.2f} "
          f"{best[12]:.2f}, slab0 issued {best[7]:.2f} us",
          flush=True)
    for o in range(4):
        cr, s0, le, ep = best[16 + 4 * o: 20 + 4 * o]
        print(f"   unit {o + 8}: C ready {cr:.2f}  slab0 {s0:.2f}  loop end {le:.2f}  epilogue {ep:.2f}  "
              f"(loop {le - s0:.2f}, epi {ep - le:.2f})",
          flush=True)
