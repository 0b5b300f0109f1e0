"""DMMA GEMM tile-config A/B (dev tool): python tools/gemm_bench.py  (LATSUM_GEMM_CFG=0..3)."""
import os, sys
import torch
sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, _lib

ctx = api.Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
shapes = [("eval_slab x16", 2048, 32768, 366, 0, 0), ("square", 8192, 8192, 8192, 0, 0),
          ("core", 366, 134000, 693, 0, 1), ("gram_tn", 1625, 1625, 4096, 1, 0)]
only = sys.argv[1] if len(sys.argv) > 1 else None
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
    for _ in range(2): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(s)
    for _ in range(reps): run()
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cfg{os.environ.get('LATSUM_GEMM_CFG','0')} {name:14s} {M}x{N}x{K}: {2*M*N*K/ms/1e9:6.2f} TF/s ({ms:.2f} ms)")
