"""Where do non-finite entries of a Tucker factor come from (dev tool)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_1411_1994_b200 import api, workload as W
from oracle import oracle as O
ctx = api.Context(0)
g = W.baseline(4)
ref = api.reference_for(g, ctx); can = api.lattice_sum(ref, g)
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
def rep_nan(tag):
    for l in range(3):
        u = t.factor(l)
        bad = ~np.isfinite(u)
        if bad.any():
            rows = np.nonzero(bad.any(axis=1))[0]; cols = np.nonzero(bad.any(axis=0))[0]
            print(tag, "mode", l, "bad", int(bad.sum()), "rows", rows.min(), rows.max(), len(rows),
                  "cols", cols.min(), cols.max(), len(cols), flush=True)
        else:
            print(tag, "mode", l, "clean", flush=True)
rep_nan("after rhosvd")
rep_nan("second download")
fx = np.load("tests/golden/fullcfg4.npz")
v = t.entries(fx["probes"]); print("probes finite", np.all(np.isfinite(v)), flush=True)
rep_nan("after tucker probes")
e = can.entries(fx["probes"]); print("canonical probes finite", np.all(np.isfinite(e)), flush=True)
rep_nan("after canonical probes")
