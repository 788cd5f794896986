"""Sub-wave problems: device time per call of the small-block kernel's
variants (strips 65..74 = variants 1..10, csrc/dgemm_small.cu) against
the persistent kernel's plans (8 = 64x32 units, 4 = 128x32 units) and the
heuristic (0), each replayed from a CUDA graph of 20 calls (device time, no
host overhead) and back-to-back from Python; every plan's C must be bitwise
the 64x32 plan's (development aid, profiles/r02/small_kernel_r02*.log).

  python tools/small_kernel_probe.py [MxNxK ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

PLANS = {0: "heur", 8: "64x32u", 4: "128x32u", 65: "s1", 66: "s2", 67: "s3", 68: "s4", 69: "s5", 70: "s6", 71: "s7",
         72: "s8", 73: "s9", 74: "s10"}
if os.environ.get("PLANS"):
    PLANS = {int(p): n for p, n in (x.split(":") for x in os.environ["PLANS"].split(","))}
shapes = [(s, s, s) for s in (128, 256, 384, 512, 640, 768, 1024, 1280)] + [
    (128, 128, 2048), (256, 256, 4096), (64, 64, 512), (17, 17, 4096), (100, 300, 1000), (200, 200, 200),
    (512, 256, 1024), (37, 53, 71), (1000, 1000, 64), (2048, 2048, 32)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
st = torch.cuda.current_stream().cuda_stream


def graph_us(fn, calls=20, reps=10):
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        fn(s2.cuda_stream)  # warm (attributes, pool) outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s2):
            for _ in range(calls):
                fn(s2.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (reps * calls))
    return best


for (m, n, k) in shapes:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c0, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    ref = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, ref.data_ptr(), m, st, strips=8)
    row = []
    for p, name in PLANS.items():
        cc = c0.clone()
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m, st, strips=p)
        torch.cuda.synchronize()
        same = torch.equal(cc, ref)
        c = c0.clone()

        def call(s, p=p, c=c):
            engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, s, strips=p)

        dev = graph_us(call)
        for _ in range(3):
            call(st)
        torch.cuda.synchronize()
        reps = max(20, int(3e6 / (m * n * k / 1e3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call(st)
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) * 1e3 / reps
        tf = 2.0 * m * n * k / dev / 1e6
        row.append(f"{name}: {dev:.2f}/{b2b:.2f} us {tf / 37.22 * 100:.1f}%{'' if same else ' MISMATCH'}")
    print(f"{m}x{n}x{k} | " + " | ".join(row), flush=True)
