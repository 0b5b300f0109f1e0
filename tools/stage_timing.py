"""Per-stage / per-kernel-class timing of the GPU pipeline on BASELINE configs (dev tool)."""
import sys, time, json
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W

cfgs = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 3]
do_eval = "--eval" in sys.argv
ctx = api.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg in cfgs:
    g = W.baseline(cfg)
    for rep_i in range(2):
        ctx.set_profiling(rep_i == 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ref = api.reference_for(g, ctx)
        can = api.lattice_sum(ref, g)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
        torch.cuda.synchronize(); t2 = time.perf_counter()
        te = 0.0
        if do_eval:
            lo, hi = g.eval_box()
            n = 1
            for a, b in zip(lo, hi): n *= (b - a)
            out = torch.empty(n, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize(); t3 = time.perf_counter()
            t.eval_box_device(lo, hi, out.data_ptr())
            torch.cuda.synchronize(); te = time.perf_counter() - t3
            del out
        print(json.dumps(dict(cfg=cfg, rep=rep_i, stage12_ms=1e3*(t1-t0), rhosvd_ms=1e3*(t2-t1),
                              eval_ms=1e3*te, ranks=rep.chosen_ranks, dict_cols=can.dict_cols,
                              T=can.merged_terms, gram=rep.gram_size, deflated=rep.deflated, k1=rep.deflate_k1,
                              margin=rep.cutoff_margin, tie=rep.tie_at_cutoff, ms=rep.ms)))
        if rep_i == 1:
            for k, v in sorted(ctx.profile().items(), key=lambda kv: -kv[1][1]):
                rate = v[2] / v[1] / 1e9 if v[1] > 0 else 0
                print(f"   {k:28s} n={v[0]:6d} ms={v[1]:10.3f} work/ms->{rate:10.2f} (TF/s or GB/s)")
        del t, can, ref
        torch.cuda.empty_cache()
