"""Dev tool: the RHOSVD spectrum of a BASELINE config against its oracle fixture, per mode,
around the cut (relative sigma error, sigma^2 error in units of the test tolerance).

    python tools/sigma_check.py 4 [LATSUM_VAR=value ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
from paper_1411_1994_b200 import api  # noqa: E402
from paper_1411_1994_b200 import workload as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
fx = np.load(os.path.join(ROOT, "tests", "golden", f"fullcfg{cfg}.npz"))
g = W.baseline(cfg)
ctx = api.Context(0)
ref = api.reference_for(g, ctx)
can = api.lattice_sum(ref, g)
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), form_core=False)
print("ranks", rep.chosen_ranks, "fixture", list(fx["ranks"]), "eig_fallbacks", ctx.eig_fallbacks)
for l in range(3):
    s_orc = fx[f"sigma{l}"]
    s_gpu = rep.singular_values[l][:s_orc.size]
    r = int(fx["ranks"][l])
    rel = np.abs(s_gpu - s_orc) / s_orc
    s2g, s2o, sr2 = s_gpu ** 2, s_orc ** 2, s_orc[r - 1] ** 2
    units = np.abs(s2g - s2o) / (2e-6 * s2o + 1e-8 * sr2)
    print(f"mode {l}: r {r} sigma_r/sigma_1 {s_orc[r - 1] / s_orc[0]:.3e}")
    for lo, hi in ((0, r - 300), (r - 300, r - 64), (r - 64, r - 8), (r - 8, r + 8), (r + 8, r + 64)):
        lo, hi = max(lo, 0), min(hi, s_orc.size)
        if hi <= lo:
            continue
        i = lo + int(np.argmax(rel[lo:hi]))
        j = lo + int(np.argmax(units[lo:hi]))
        print(f"   [{lo:5d},{hi:5d}) max rel {rel[i]:.2e} at {i} (s/s1 {s_orc[i] / s_orc[0]:.2e}); "
              f"max tol units {units[j]:.2f} at {j}")
    tail_g = np.sqrt(np.sum(rep.singular_values[l][r:] ** 2))
    tail_o = np.sqrt(np.sum(s_orc[r:] ** 2))
    print(f"   tail rel {abs(tail_g - tail_o) / tail_o:.2e}")
