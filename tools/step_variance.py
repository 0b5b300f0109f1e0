"""Per-step stage times of the bench loop (flush + stages 1-3 + evaluation), to locate
step-time outliers (dev tool).  python tools/step_variance.py CFG STEPS [--no-eval] [--no-smi]"""
import json, subprocess, sys, time
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W
cfg, steps = int(sys.argv[1]), int(sys.argv[2])
g = W.baseline(cfg)
ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
lo, hi = g.eval_box()
n = (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2])
do_eval = "--no-eval" not in sys.argv
out = torch.empty(n if do_eval else 1, dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
smi = None if "--no-smi" in sys.argv else subprocess.Popen(
    ["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader", "-lms", "200"],
    stdout=subprocess.DEVNULL)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
prof = "--prof" in sys.argv
ctx.set_profiling(prof)
for i in range(steps):
    flush.zero_(); torch.cuda.synchronize()
    ev[0].record(s)
    ref = api.reference_for(g, ctx); can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    ev[1].record(s)
    if do_eval:
        t.eval_box_device(lo, hi, out.data_ptr())
    ev[2].record(s); torch.cuda.synchronize()
    free, _ = torch.cuda.mem_get_info()
    print(json.dumps(dict(step=i, ms13=round(ev[0].elapsed_time(ev[1]), 1),
                          eval=round(ev[1].elapsed_time(ev[2]), 1),
                          ms={k: round(v, 1) for k, v in rep.ms.items()},
                          free_gb=round(free / 2**30, 1))), flush=True)
    if prof:
        p = ctx.profile()
        top = sorted(p.items(), key=lambda kv: -kv[1][1])[:8]
        print("   ", {k: (v[0], round(v[1], 1)) for k, v in top}, flush=True)
        ctx.set_profiling(False); ctx.set_profiling(True)
    del t, can, ref
if smi:
    smi.terminate()
