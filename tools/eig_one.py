"""One two-stage eigensolve at size n (dev tool for ncu captures of the band kernels)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1411_1994_b200 import _lib, api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 693
method = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = api.Context(0)
rng = np.random.default_rng(n)
Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
A = (Q * 10.0 ** (-16 * np.arange(n) / (n - 1))) @ Q.T
dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
k = n // 2
w = torch.zeros(n, dtype=torch.float64, device="cuda")
V = torch.zeros(n * k, dtype=torch.float64, device="cuda")
ctx.check(_lib.lib().latsum_eig_sym_device(ctx.handle, n, dA.data_ptr(), k, w.data_ptr(), V.data_ptr(), method))
torch.cuda.synchronize()
print("ok", w[-3:].cpu().numpy())
