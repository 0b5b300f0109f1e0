"""Oracle fixtures for the full-size BASELINE configs 2-5 (run here; ~10 min for cfg5):

    python tests/golden/make_fullconfig.py [cfg ...]

Writes fullcfg<i>.npz: RHOSVD ranks / tie flags / cut-off margins and the leading
singular values per mode (column-merged LAPACK SVD of the oracle's side matrices),
weight and input norms, and at seeded probes the RHOSVD reconstruction
(projected-CP identity), the untruncated canonical value and (on a subset) the
brute-force windowed-sum oracle (lattice_sum.hpp:656-671)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1411_1994_b200 import workload as W  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N_PROBES, N_BRUTE = 500, 100  # cmd_verify: 500 probes (commands.cpp:254-266)


def make(cfg: int):
    t0 = time.time()
    g = W.baseline(cfg)
    ref = O.reference(g)
    sides, w = O.side_dictionary(ref, g)
    orc = O.rhosvd(sides, w, eps=g.eps, with_norm=True)
    pr = O.probes(g.N, N_PROBES, 1000 + cfg)
    lo, hi = g.eval_box()
    # half the probes inside the evaluation box
    inbox = np.stack([np.random.default_rng(cfg).integers(lo[l], hi[l], N_PROBES // 2)
                      for l in range(3)], axis=1)
    pr = np.concatenate([pr[:N_PROBES // 2], inbox]).astype(np.int64)
    v_rhosvd = O.projected_cp_entries(w, orc.Z, orc.P, pr)
    v_canon = O.canonical_entries(sides, w, pr)
    v_brute = O.oracle_entries(ref, g, pr[:N_BRUTE])
    keep = [min(orc.sigma[l].size, orc.ranks[l] + 512) for l in range(3)]
    np.savez_compressed(
        os.path.join(HERE, f"fullcfg{cfg}.npz"),
        ranks=np.array(orc.ranks), tie=np.array(orc.tie), margin=np.array(orc.margin),
        sigma0=orc.sigma[0][:keep[0]], sigma1=orc.sigma[1][:keep[1]], sigma2=orc.sigma[2][:keep[2]],
        n_singular=np.array([s.size for s in orc.sigma]),
        weight_norm=orc.weight_norm, input_norm=orc.input_norm, bound_abs=orc.bound_abs,
        probes=pr, v_rhosvd=v_rhosvd, v_canonical=v_canon, v_brute=v_brute, C0=ref.C0,
        canonical_rank=w.size, merged_columns=np.array([sd.U.shape[1] for sd in sides]))
    print(f"cfg{cfg}: ranks {orc.ranks} margins {orc.margin} ties {orc.tie} "
          f"brute-vs-canonical {np.max(np.abs(v_brute - v_canon[:N_BRUTE])) / np.max(np.abs(v_brute)):.2e} "
          f"({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["2", "3", "4", "5"]):
        make(int(c))
