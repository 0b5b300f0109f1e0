"""Timing of the custom eigensolver stages vs cuSOLVER syevd at the Gram sizes (dev tool)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, _lib

ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
L = _lib.lib()
for n in [int(a) for a in sys.argv[1:]] or [357, 693, 1625]:
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n, n))
    A0 = torch.from_numpy(np.asfortranarray(B @ B.T).ravel(order="F").copy()).cuda()
    A = A0.clone()
    d = torch.zeros(n, dtype=torch.float64, device="cuda")
    e = torch.zeros(n, dtype=torch.float64, device="cuda")
    tau = torch.zeros(n, dtype=torch.float64, device="cuda")
    def run():
        A.copy_(A0)
        ctx.check(L.latsum_sytrd_device(ctx.handle, n, A.data_ptr(), n, d.data_ptr(), e.data_ptr(),
                                        tau.data_ptr()))
    for _ in range(2): run()
    ctx.set_profiling(True)
    for _ in range(5): run()
    torch.cuda.synchronize()
    prof = ctx.profile()
    ctx.set_profiling(False)
    print(f"n={n}: " + ", ".join(f"{k} {v[1] / v[0]:.3f} ms" for k, v in prof.items()), flush=True)
