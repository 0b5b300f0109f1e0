"""cfg5 stages 1-3 (factors-only RHOSVD) then a 2048 x 2048 x 32 box of the central
evaluation inside an NVTX range 'eval', for ncu captures of the assembly kernels (NVTX range
'assemble') and the grouped projected-CP evaluation kernels (dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W

ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
g = W.baseline(5)
ref = api.reference_for(g, ctx)
torch.cuda.nvtx.range_push("assemble")
can = api.lattice_sum(ref, g)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), form_core=False)
c = g.N[0] // 2
lo, hi = (c - 1024, c - 1024, c - 16), (c + 1024, c + 1024, c + 16)
out = torch.empty(2048 * 2048 * 32, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("eval")
t.eval_box_device(lo, hi, out.data_ptr())
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ranks", rep.chosen_ranks, "sum", float(out.sum()))
