"""Fixed vs per-k cost of small problems (development aid): device time of
one call for m = n in {256, 512, 1024} and growing k, next to an empty
torch kernel launch (the event-to-event floor)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine


def best_of(fn, reps=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[0], ts[len(ts) // 2]


x = torch.zeros(1, device="cuda")
print("empty launch (x.add_(1)): best %.2f us median %.2f us" % best_of(lambda: x.add_(1)), flush=True)
st = torch.cuda.current_stream().cuda_stream
strips = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--strips=")]
for mn in (256, 512, 1024):
    for k in (16, 64, 256, 512, 1024, 2048):
        a = torch.empty(mn * k, dtype=torch.float64, device="cuda")
        b = torch.empty(k * mn, dtype=torch.float64, device="cuda")
        c = torch.empty(mn * mn, dtype=torch.float64, device="cuda")
        for t, (buf, r, cc) in enumerate(((a, mn, k), (b, k, mn), (c, mn, mn))):
            engine.fill_random_device(buf.data_ptr(), r, cc, r, 7 + t, 0, st)
        for s in strips or [0]:
            bst, med = best_of(lambda: engine.dgemm_device(mn, mn, k, a.data_ptr(), mn, b.data_ptr(), k,  # noqa: B023
                                                           c.data_ptr(), mn, st, strips=s))
            print(f"{mn}x{mn}x{k} strips={s}: best {bst:.2f} us median {med:.2f} us "
                  f"{2 * mn * mn * k / bst / 1e6:.2f} TF", flush=True)
