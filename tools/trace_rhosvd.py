"""Host timeline of one cfg2 pipeline (LATSUM_TRACE=1), after warm-up (dev tool)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W
ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
g = W.baseline(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for i in range(3):
    t0 = time.perf_counter()
    ref = api.reference_for(g, ctx); torch.cuda.synchronize(); t1 = time.perf_counter()
    can = api.lattice_sum(ref, g); torch.cuda.synchronize(); t2 = time.perf_counter()
    if i == 2:
        print(f"--- step {i}: reference {1e3*(t1-t0):.2f} ms, assembly {1e3*(t2-t1):.2f} ms", file=sys.stderr, flush=True)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps)); torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"step {i}: ref {1e3*(t1-t0):.2f} asm {1e3*(t2-t1):.2f} rhosvd {1e3*(t3-t2):.2f} ms", file=sys.stderr, flush=True)
