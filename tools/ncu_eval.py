"""Small stage-1..4 run of cfg2 for ncu captures: the evaluation box is 2048 x 2048 x 64
(one z-chunk) and is wrapped in an NVTX range 'eval' so `ncu --nvtx --nvtx-include eval/`
can select its kernels (Q GEMM, X GEMM, slab GEMM).  Dev tool."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W

ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
g = W.baseline(2)
ref = api.reference_for(g, ctx)
can = api.lattice_sum(ref, g)
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
lo, hi = (0, 0, 0), (2048, 2048, 64)
out = torch.empty(2048 * 2048 * 64, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("eval")
t.eval_box_device(lo, hi, out.data_ptr())
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ranks", rep.chosen_ranks, "sum", float(out.sum()))
