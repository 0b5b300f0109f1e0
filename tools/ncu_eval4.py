"""cfg4 stages 1-3, then the central 2048 x 2048 x 64 z-slab of the evaluation box inside an
NVTX range 'eval' (`ncu --nvtx --nvtx-include eval/` selects its kernels: core slicing, Q, X
and slab GEMMs).  Dev tool for the round's ncu captures."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W

ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
g = W.baseline(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
ref = api.reference_for(g, ctx)
can = api.lattice_sum(ref, g)
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
lo, hi = g.eval_box()
lo2, hi2 = lo, (hi[0], hi[1], lo[2] + 64)
out = torch.empty(2048 * 2048 * 64, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("eval")
t.eval_box_device(lo2, hi2, out.data_ptr())
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ranks", rep.chosen_ranks, "sum", float(out.sum()))
