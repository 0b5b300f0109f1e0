"""Device->host copy bandwidth into pinned memory, 1 vs 2 streams (dev tool)."""
import torch
n = 4 * 2**30 // 8
d = torch.ones(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:
        s.wait_event(e0)
    part = n // ns
    for q, s in enumerate(ss):
        with torch.cuda.stream(s):
            h[q * part:(q + 1) * part].copy_(d[q * part:(q + 1) * part], non_blocking=True)
    for s in ss:
        e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    print(ns, "streams", round(n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), "GB/s")
