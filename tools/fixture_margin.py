"""Print the reconstruction error of each full-config fixture relative to its 10 eps + 1e-12
tolerance (dev tool: margin check for numerics changes)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1411_1994_b200 import api, workload as W  # noqa: E402

ctx = api.Context(0)
for cfg in [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]:
    fx = np.load(os.path.join("tests", "golden", f"fullcfg{cfg}.npz"))
    g = W.baseline(cfg)
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), form_core=(cfg != 5))
    v = t.entries(fx["probes"])
    want = fx["v_rhosvd"]
    err = np.max(np.abs(v - want)) / np.max(np.abs(want))
    s_err = max(np.max(np.abs(rep.singular_values[l][:fx[f"sigma{l}"].size] - fx[f"sigma{l}"]))
                / fx[f"sigma{l}"][0] for l in range(3))
    print(f"cfg{cfg}: ranks {rep.chosen_ranks} vs {list(fx['ranks'])}, value err {err:.3e} "
          f"(tol {10 * g.eps + 1e-12:.1e}, ratio {err / (10 * g.eps + 1e-12):.3f}), sigma err {s_err:.2e}",
          flush=True)
