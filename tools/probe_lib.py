"""One-off probe: cuBLAS DGEMM yardstick and cuSOLVER syevd timings (via torch). Not product code."""
import time, torch
dev = "cuda"
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    ms = t(lambda: a @ b)
    print(f"DGEMM {n}: {2*n**3/ms/1e9:.2f} TFLOP/s")
a = torch.randn(2048, 40000, dtype=torch.float64, device=dev)
ms = t(lambda: a @ a.T)
print(f"DGEMM AAT 2048x40000: {2*2048*2048*40000/ms/1e9:.2f} TFLOP/s {ms:.2f} ms")
for n in (512, 1024, 2048, 4096, 8192):
    x = torch.randn(n, n, dtype=torch.float64, device=dev); x = x + x.T
    ms = t(lambda: torch.linalg.eigh(x), reps=2)
    ms2 = t(lambda: torch.linalg.eigvalsh(x), reps=2)
    print(f"eigh {n}: {ms:.1f} ms   eigvalsh {ms2:.1f} ms")
