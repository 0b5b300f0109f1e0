import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, _lib
M, N, K = [int(a) for a in sys.argv[1:4]]
ctx = api.Context(0)
rng = np.random.default_rng(0)
A = rng.standard_normal((M, K)); B = rng.standard_normal((K, N))
dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F")).cuda()
dB = torch.from_numpy(np.asfortranarray(B).ravel(order="F")).cuda()
dC = torch.zeros(M * N, dtype=torch.float64, device="cuda")
ctx.check(_lib.lib().latsum_dgemm_ozaki_device(ctx.handle, 0, M, N, K, dA.data_ptr(), M, dB.data_ptr(), K, dC.data_ptr(), M))
ctx.synchronize()
got = dC.cpu().numpy().reshape((M, N), order="F")
print(M, N, K, "max err", np.max(np.abs(got - A @ B)))
