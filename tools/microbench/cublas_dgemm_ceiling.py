"""One-off probe: cuBLAS DGEMM rate via torch (a ceiling reference only; never on the product path)."""
import torch, time, subprocess
torch.backends.cuda.matmul.allow_tf32 = False
for n in (2048, 4096, 8192):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    c = torch.rand(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c.addmm_(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        c.addmm_(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cublas dgemm n={n}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} GFLOP/s")
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
