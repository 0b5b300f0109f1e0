import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, _lib
n = int(sys.argv[1])
ctx = api.Context(0)
rng = np.random.default_rng(n)
B = rng.standard_normal((n, n)); A = (B + B.T) / 2
dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
d = torch.zeros(n, dtype=torch.float64, device="cuda"); e = torch.zeros(max(n-1,1), dtype=torch.float64, device="cuda"); t = torch.zeros(max(n-1,1), dtype=torch.float64, device="cuda")
st = _lib.lib().latsum_sytrd_device(ctx.handle, n, dA.data_ptr(), n, d.data_ptr(), e.data_ptr(), t.data_ptr())
print(n, "status", st, _lib.lib().latsum_last_error(ctx.handle))
try:
    ctx.synchronize()
    T = np.diag(d.cpu().numpy()) + np.diag(e.cpu().numpy()[:n-1], 1) + np.diag(e.cpu().numpy()[:n-1], -1)
    print(n, "eig err", np.max(np.abs(np.linalg.eigvalsh(T) - np.linalg.eigvalsh(A))))
except Exception as ex:
    print(n, "sync error", ex)
