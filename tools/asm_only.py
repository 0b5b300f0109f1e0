"""Stages 1-2 (reference tensor + dictionary assembly) of one BASELINE config, for ncu
captures of the assembly kernels (dev tool)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W  # noqa: E402

ctx = api.Context(0)
g = W.baseline(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
for _ in range(2):
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    torch.cuda.synchronize()
print("ok", can.dict_cols)
