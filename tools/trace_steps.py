"""Host timeline (LATSUM_TRACE=1) of several cfg-N RHOSVD steps, to find step-time variance (dev tool)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W
ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
g = W.baseline(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
do_eval = "--eval" in sys.argv
lo, hi = g.eval_box()
n = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2])
out = torch.empty(n if do_eval else 1, dtype=torch.float64, device="cuda")
for i in range(steps):
    torch.cuda.synchronize()
    print(f"=== step {i}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps)); torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    print(f"=== step {i} total {1e3*(time.perf_counter()-t0):.1f} ms (free {free/2**30:.1f} GiB)", file=sys.stderr, flush=True)
    if do_eval:
        t1 = time.perf_counter()
        t.eval_box_device(lo, hi, out.data_ptr()); torch.cuda.synchronize()
        free, total = torch.cuda.mem_get_info()
        print(f"=== step {i} eval {1e3*(time.perf_counter()-t1):.1f} ms, free {free/2**30:.1f} GiB", file=sys.stderr, flush=True)
    del t, can, ref
