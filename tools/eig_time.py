"""Time the symmetric eigensolver backends (cuSOLVER syevd, one-stage cluster sytrd,
two-stage band) on Gram-like matrices at the RHOSVD sizes, plus a per-kernel profile of the
two-stage path (dev tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1411_1994_b200 import _lib, api  # noqa: E402

ctx = api.Context(0)
L = _lib.lib()
sizes = [int(a) for a in sys.argv[1:]] or [357, 693, 800]
for n in sizes:
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-16 * np.arange(n) / (n - 1))
    A = (Q * lam) @ Q.T
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
    k = n // 2
    w = torch.zeros(n, dtype=torch.float64, device="cuda")
    V = torch.zeros(n * k, dtype=torch.float64, device="cuda")
    for method in [1, 2, 3]:
        ts = []
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx.check(L.latsum_eig_sym_device(ctx.handle, n, dA.data_ptr(), k, w.data_ptr(),
                                              V.data_ptr(), method))
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"n={n} k={k} method={method}: best {min(ts):.2f} ms  {['%.2f' % t for t in ts]}",
              flush=True)
    ctx.set_profiling(True)
    ctx.check(L.latsum_eig_sym_device(ctx.handle, n, dA.data_ptr(), k, w.data_ptr(), V.data_ptr(), 3))
    torch.cuda.synchronize()
    for tag, (cnt, ms, _) in sorted(ctx.profile().items(), key=lambda x: -x[1][1]):
        print(f"    {tag:24s} {cnt:4d} {ms:8.3f} ms")
    ctx.set_profiling(False)
