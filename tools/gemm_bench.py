"""DMMA GEMM tile-config A/B (dev tool): python tools/gemm_bench.py [shape-prefix] [--ozaki]
(LATSUM_GEMM_CFG=0..3 selects the DMMA tile; --ozaki times the int8 tensor-core GEMM on the
NN shapes as well, split into slicing and the tcgen05 kernel via the profiling scopes)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, _lib

ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
shapes = [("eval_slab x16", 2048, 32768, 366, 0, 0), ("eval_slab x64", 2048, 131072, 384, 0, 0),
          ("square", 8192, 8192, 8192, 0, 0),
          ("core", 366, 134000, 693, 0, 1), ("gram_tn", 1625, 1625, 4096, 1, 0)]
args = [a for a in sys.argv[1:] if not a.startswith("--")]
ozaki = "--ozaki" in sys.argv
only = args[0] if args else None
for name, M, N, K, ta, tb in shapes:
    if only and not name.startswith(only):
        continue
    A = torch.randn(M * K, dtype=torch.float64, device="cuda")
    B = torch.randn(K * N, dtype=torch.float64, device="cuda")
    C = torch.empty(M * N, dtype=torch.float64, device="cuda")
    lda = K if ta else M
    ldb = N if tb else K
    def run():
        ctx.check(_lib.lib().latsum_dgemm_device(ctx.handle, ta, tb, M, N, K, 1.0, A.data_ptr(), lda,
                                                 B.data_ptr(), ldb, 0.0, C.data_ptr(), M))
    def run_oz():
        ctx.check(_lib.lib().latsum_dgemm_ozaki_device(ctx.handle, 0, M, N, K, A.data_ptr(), M,
                                                       B.data_ptr(), K, C.data_ptr(), M))
    variants = [("dmma", run)] + ([("ozaki", run_oz)] if ozaki and not ta and not tb else [])
    for vname, fn in variants:
        for _ in range(2): fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        ctx.set_profiling(True)
        e0.record(s)
        for _ in range(reps): fn()
        e1.record(s); torch.cuda.synchronize()
        prof = ctx.profile()
        ctx.set_profiling(False)
        ms = e0.elapsed_time(e1) / reps
        parts = ", ".join(f"{k} {v[1] / reps:.2f} ms" for k, v in prof.items())
        print(f"{vname} cfg{os.environ.get('LATSUM_GEMM_CFG','0')} {name:14s} {M}x{N}x{K}: "
              f"{2*M*N*K/ms/1e9:6.2f} TF/s ({ms:.2f} ms) [{parts}]")
