"""Full-box evaluation of a BASELINE config: NaN / inf count per z-slice (dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W
ctx = api.Context(0)
g = W.baseline(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
ref = api.reference_for(g, ctx); can = api.lattice_sum(ref, g)
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
lo, hi = g.eval_box()
ni, nj, nk = (hi[l] - lo[l] for l in range(3))
for trial in range(2):
    if "--trim" in sys.argv:
        ctx.trim_pool()
    torch.cuda.synchronize()
    out = torch.empty(ni * nj * nk, dtype=torch.float64, device="cuda")
    out.fill_(float("nan"))
    t.eval_box_device(lo, hi, out.data_ptr())
    ctx.synchronize()
    v = out.view(nk, nj, ni)
    nz, tot = [], 0
    for k0 in range(0, nk, 32):
        b = (~torch.isfinite(v[k0:k0 + 32])).sum(dim=(1, 2))
        tot += int(b.sum())
        nz += [k0 + i for i in torch.nonzero(b).flatten().tolist()]
    print("trial", trial, "bad slices", len(nz), nz[:10], "total bad", tot, flush=True)
    del out, v
    torch.cuda.empty_cache()
