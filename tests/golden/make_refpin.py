"""Golden vectors from the REFERENCE ITSELF (run in the build container, where /root/reference
exists):

    python tests/golden/make_refpin.py [case ...]

oracle/_ref/liblatsum_ref.so is the reference's own headers compiled where they lie against the
stand-ins of oracle/shim (oracle/Makefile `ref`); oracle/ref.py drives it.  For every case in
`oracle.ref.CASES` (geometries the reference API can express) this writes refpin_<case>.npz:

* stage 1: calibrated C0, nodes, quadrature weights, the 2N x R reference side matrix per
  distinct mode and its weights (build_reference_canonical, reference.hpp:95-153);
* stage 2: the N x M_c side matrices (columns F_cols: all of them, every 16th for M_c > 512) and weights of the canonical sum in the reference's term
  order (assembled_sum_canonical / sublattice_union_sum / defected_sum,
  lattice_sum.hpp:198-223, 411-465, 339-384) and its provenance summands;
* stage 3: rhosvd ranks, tie flags, singular values and report (rank_reduction.hpp:176-218),
  canonical_to_tucker ranks after 3 ALS sweeps (rank_reduction.hpp:280-306);
* stage 4: Tucker / canonical entries at seeded probes (tucker.hpp:38-54, canonical.hpp:63-70)
  and the brute-force oracle_entry (lattice_sum.hpp:656-672) on a subset;
* (case "cubic") the bytes of the reference's own tensor files (write_tensor, src/tensor_io.cpp).

The GPU box has no /root/reference: tests read these files there.  tests/test_reference_pin.py
re-derives them from the live library whenever it is present, so they cannot go stale."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref as RF  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N_PROBES, N_BRUTE, C2T_SWEEPS = 200, 40, 3


def probes(dims, count, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.stack([rng.integers(0, dims[l], count) for l in range(3)], axis=1).astype(np.int64)


def derive(name: str) -> dict:
    """Everything the fixture holds, from one live reference run."""
    c = RF.CASES[name]
    r = RF.RefRun(name)
    try:
        rr = r.reference()
        r.sum()
        F, w = r.canonical()
        summ = r.summands()
        red = r.reduce("rhosvd", eps=c["eps"])
        pr = probes(rr["N"], N_PROBES, 77)
        v_t = r.entries("tucker", pr)
        v_c = r.entries("canonical", pr)
        v_b = r.entries("oracle", pr[:N_BRUTE])
        files = {}
        if name == "cubic":  # the reference's own tensor files (write_tensor, src/tensor_io.cpp)
            import tempfile
            with tempfile.TemporaryDirectory() as td:
                r.write_tensor("canonical", os.path.join(td, "c.tns"))
                r.write_tensor("tucker", os.path.join(td, "t.tns"))
                files["tensor_file_canonical"] = np.frombuffer(open(os.path.join(td, "c.tns"), "rb").read(), np.uint8)
                files["tensor_file_tucker"] = np.frombuffer(open(os.path.join(td, "t.tns"), "rb").read(), np.uint8)
        if c.get("c2t", True):
            c2t = r.reduce("c2t", eps=c["eps"], max_als_sweeps=C2T_SWEEPS)
            v_c2t = r.entries("tucker", pr)
        else:
            c2t, v_c2t = dict(ranks=()), np.zeros(0)
    finally:
        r.close()
    # large cases keep every 16th column of the side matrices (F_cols), small ones all
    cols = np.arange(w.size) if w.size <= 512 else np.arange(0, w.size, 16)
    out = dict(
        N=np.array(rr["N"]), C0=rr["C0"], shell=np.array(rr["shell"]), nodes=rr["nodes"],
        quad_weights=rr["quad_weights"], ref_weights=rr["weights"],
        ref_factor0=rr["factors"][0], ref_factor1=rr["factors"][1], ref_factor2=rr["factors"][2],
        F0=F[0][:, cols], F1=F[1][:, cols], F2=F[2][:, cols], F_cols=cols, weights=w,
        summand_labels=np.array([s[0] for s in summ]), summand_ranks=np.array([s[1] for s in summ]),
        summand_sites=np.array([s[2] for s in summ]),
        ranks=np.array(red["ranks"]), ties=np.array(red["ties"]),
        sv0=red["sv"][0], sv1=red["sv"][1], sv2=red["sv"][2],
        report=np.array([red["bound_abs"], red["bound_rel"], red["weight_norm"], red["input_norm"],
                         red["stability_constant"], float(red["stability_ok"])]),
        probes=pr, v_tucker=v_t, v_canonical=v_c, v_brute=v_b,
        c2t_ranks=np.array(c2t["ranks"], np.int64), v_c2t=v_c2t, c2t_sweeps=C2T_SWEEPS, **files)
    return out


def make(name: str):
    t0 = time.time()
    d = derive(name)
    np.savez_compressed(os.path.join(HERE, f"refpin_{name}.npz"), **d)
    print(f"{name}: N {d['N'].tolist()} M_c {d['weights'].size} ranks {d['ranks'].tolist()} "
          f"c2t {d['c2t_ranks'].tolist()} ties {d['ties'].tolist()} ({time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    if not RF.build():
        raise SystemExit("oracle/_ref is not built and /root/reference is absent")
    for name in (sys.argv[1:] or list(RF.CASES)):
        make(name)
