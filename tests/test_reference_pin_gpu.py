"""GPU parity against the REFERENCE ITSELF: the CUDA path (through the C ABI) against outputs of
the reference's own code (tests/golden/refpin_*.npz, written by tests/golden/make_refpin.py from
oracle/_ref = /root/reference/proj compiled against the stand-ins of oracle/shim; kept current by
tests/test_reference_pin.py).  Same bars as test_parity_gpu.py: unit side-matrix columns 1e-12,
identical RHOSVD ranks, singular values 1e-10 sigma_1, reconstructed potentials within
10 eps + 1e-12 of the exact sum and 1e-9 of the reference's own truncated values."""
import os
import re

import numpy as np
import pytest

from oracle import ref as RF
from paper_1411_1994_b200 import api
from latsum_helpers import col_rel_linf

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = RF.single_kernel_cases()


def fixture(name):
    return np.load(os.path.join(GOLD, f"refpin_{name}.npz"))


@pytest.mark.parametrize("name", CASES)
def test_cuda_path_reproduces_the_reference(ctx, name):
    fx = fixture(name)
    g = RF.geometry(name)
    # ---- stage 1 (build_reference_canonical, reference.hpp:95-153)
    ref = api.reference_for(g, ctx)
    assert ref.step_constant == float(fx["C0"])
    t, a = ref.quadrature()
    assert np.array_equal(t, fx["nodes"]) and np.array_equal(a, fx["quad_weights"])
    for l in range(3):
        assert col_rel_linf(ref.factor(l), fx[f"ref_factor{l}"]) < 1e-12
    np.testing.assert_allclose(ref.weights, fx["ref_weights"], rtol=1e-13)
    # ---- stage 2 (assembled_sum_canonical / sublattice_union_sum / defected_sum): the
    # reference's term order, columns and weights
    can = api.lattice_sum(ref, g)
    assert can.rank == fx["weights"].size
    cols = fx["F_cols"]
    for l in range(3):
        assert col_rel_linf(can.factor(l)[:, cols], fx[f"F{l}"]) < 1e-12
    np.testing.assert_allclose(can.weights, fx["weights"], rtol=1e-12,
                               atol=1e-15 * np.abs(fx["weights"]).max())
    # ---- stage 3 (rhosvd, rank_reduction.hpp:176-218)
    tk, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    assert tuple(rep.chosen_ranks) == tuple(int(x) for x in fx["ranks"])
    assert tk.ranks == rep.chosen_ranks
    for l in range(3):
        sv = fx[f"sv{l}"]
        assert rep.singular_values[l].size == sv.size
        assert np.max(np.abs(rep.singular_values[l] - sv)) <= 1e-10 * sv[0]
    bound_abs, bound_rel, weight_norm, input_norm, stab, stab_ok = fx["report"]
    np.testing.assert_allclose(rep.weight_norm, weight_norm, rtol=1e-12)
    np.testing.assert_allclose(rep.input_norm, input_norm, rtol=1e-9)
    np.testing.assert_allclose(rep.stability_constant, stab, rtol=1e-8)
    assert rep.stability_ok == bool(stab_ok)
    np.testing.assert_allclose(rep.bound_abs, bound_abs, rtol=1e-3,
                               atol=1e-12 * weight_norm * fx["sv0"][0])
    # ---- stage 4 (TuckerTensor::entry, CanonicalTensor::entry, oracle_entry)
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    assert np.max(np.abs(can.entries(pr) - fx["v_canonical"])) <= 1e-12 * scale
    v = tk.entries(pr)
    assert np.max(np.abs(v - fx["v_canonical"])) <= (10 * g.eps + 1e-12) * scale
    assert np.max(np.abs(v - fx["v_tucker"])) <= 1e-9 * scale  # the reference's truncated values
    nb = fx["v_brute"].size
    assert np.max(np.abs(api.oracle_entries(ref, g, pr[:nb]) - fx["v_brute"])) <= 1e-12 * scale


@pytest.mark.parametrize("name", ["vacancies", "yukawa", "union", "clusters"])
def test_cuda_canonical_to_tucker_matches_the_reference(ctx, name):
    """canonical_to_tucker (rank_reduction.hpp:280-306) after 3 ALS sweeps: the reference's ranks
    (+-1 where a slice-drop decision sits within 5% of the budget, whose own cancellation noise is
    percent level) and values within the tolerance of the exact sum and 3 eps of the reference's
    (two truncations at eps ||A|| each)."""
    fx = fixture(name)
    g = RF.geometry(name)
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep, sweeps = api.canonical_to_tucker(can, api.TruncationSpec.tol(g.eps),
                                             max_als_sweeps=int(fx["c2t_sweeps"]))
    want = tuple(int(x) for x in fx["c2t_ranks"])
    assert all(abs(rep.chosen_ranks[l] - want[l]) <= 1 for l in range(3)), (rep.chosen_ranks, want)
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    got = t.entries(pr)
    assert np.max(np.abs(got - fx["v_canonical"])) <= 30 * g.eps * scale
    if tuple(rep.chosen_ranks) == want:
        assert np.max(np.abs(got - fx["v_c2t"])) <= 3 * g.eps * scale


def test_cuda_path_reads_the_references_tensor_files(ctx, tmp_path):
    """latsum_tensor_read on files the reference itself wrote (write_tensor, src/tensor_io.cpp):
    same entries as the reference evaluates from them, and a tampered file is rejected."""
    fx = fixture("cubic")
    pc, pt = tmp_path / "c.tns", tmp_path / "t.tns"
    pc.write_bytes(fx["tensor_file_canonical"].tobytes())
    pt.write_bytes(fx["tensor_file_tucker"].tobytes())
    can = api.read_tensor(pc, ctx)
    tk = api.read_tensor(pt, ctx)
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    assert can.rank == fx["weights"].size and tuple(tk.ranks) == tuple(int(x) for x in fx["ranks"])
    assert np.max(np.abs(can.entries(pr) - fx["v_canonical"])) <= 1e-13 * scale
    assert np.max(np.abs(tk.entries(pr) - fx["v_tucker"])) <= 1e-13 * scale
    # re-writing what was read reproduces the reference's bytes
    api.write_tensor(tmp_path / "c2.tns", can)
    api.write_tensor(tmp_path / "t2.tns", tk)
    assert (tmp_path / "c2.tns").read_bytes() == pc.read_bytes()
    assert (tmp_path / "t2.tns").read_bytes() == pt.read_bytes()
    raw = bytearray(pt.read_bytes())
    raw[50] ^= 0x10
    pt.write_bytes(bytes(raw))
    with pytest.raises(IOError):
        api.read_tensor(pt, ctx)


@pytest.mark.parametrize("name", ["cubic", "vacancies", "yukawa", "clusters", "active", "large"])
def test_references_own_verify_accepts_the_cuda_results(ctx, name, tmp_path):
    """The reference's own `latsum verify` (cmd_verify, src/commands.cpp:200-284, run from
    oracle/_ref) on tensor files the CUDA path wrote: it reads them (checksum-guarded), enumerates
    the sources of the same geometry, and checks 500 mt19937_64 probes against its brute-force
    oracle — the canonical sum at its default tolerance 1e-10, the RHOSVD result against the
    truncation bound recorded in the provenance sidecar the CUDA path wrote."""
    if not RF.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    g = RF.geometry(name)
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    tk, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    pc, pt, pp = tmp_path / "c.tns", tmp_path / "t.tns", tmp_path / "p.txt"
    api.write_tensor(pc, can)
    api.write_tensor(pt, tk)
    api.write_provenance(str(pp), g, tk, rep, seed=9)
    r = RF.RefRun(name)
    try:
        r.sum()  # the handle's geometry now carries the case's defects
        ok, log, err = r.cmd_verify(pc, None, probes=500, tolerance=1e-10, seed=9)
        assert ok and log.rstrip().endswith("verify: ok"), (log, err)
        # (an untruncated result records the bound 0 here: the merged-column Gram has exact zeros
        # where the reference's SVD leaves ~1e-16 sigma_1 noise; the bound gate needs a real tail)
        if rep.bound_abs > 1e-12 * rep.weight_norm * rep.singular_values[0][0]:
            ok, log, err = r.cmd_verify(pt, pp, probes=500, seed=9)
            assert ok and "within bound" in log, (log, err)
        # and at the reference's own normalised-error gate for a truncated result
        ok, log, err = r.cmd_verify(pt, None, probes=500, tolerance=10 * g.eps, seed=9)
        assert ok, (log, err)
        # api.verify (device brute force, latsum_verify_probes) visits the probes cmd_verify visits
        # for the same seed and measures what it measures
        m = re.search(r"max abs error (\S+), max \|oracle\| (\S+), normalized error (\S+)", log)
        ref_abs, ref_mag, ref_rel = (float(m.group(i).rstrip(",")) for i in (1, 2, 3))
        mine = api.verify(tk, ref, g, probes=500, seed=9, tolerance=10 * g.eps)
        assert mine["ok"] and mine["probes"] == 500
        np.testing.assert_allclose(mine["max_oracle"], ref_mag, rtol=1e-12)
        np.testing.assert_allclose(mine["max_abs"], ref_abs, rtol=1e-3, atol=1e-13 * ref_mag)
    finally:
        r.close()


def test_cuda_path_per_defect_kernels_match_the_reference(ctx):
    """DefectSpec.kernel: a Newton lattice with Newton vacancies and Yukawa impurity clusters,
    interleaved.  Each run of same-kernel defects is assembled against that kernel's reference
    tensor and added with latsum_canonical_concat (add_concat, canonical.hpp:94-110) in DefectSpec
    order, as defected_sum does (lattice_sum.hpp:355-378); the result is the reference's: term
    order, columns, weights, RHOSVD ranks, values, and the brute-force sum over both kernels."""
    fx = fixture("mixed_kernels")
    total = None
    for fam, lam, g in RF.geometry_parts("mixed_kernels"):
        part = api.lattice_sum(api.reference_for(g, ctx), g)
        total = part if total is None else api.add_concat(total, part)
    assert total.rank == fx["weights"].size == 105
    cols = fx["F_cols"]
    for l in range(3):
        assert col_rel_linf(total.factor(l)[:, cols], fx[f"F{l}"]) < 1e-12
    np.testing.assert_allclose(total.weights, fx["weights"], rtol=1e-12)
    eps = RF.CASES["mixed_kernels"]["eps"]
    tk, rep = api.rhosvd(total, api.TruncationSpec.tol(eps))
    assert tuple(rep.chosen_ranks) == tuple(int(x) for x in fx["ranks"])
    for l in range(3):
        assert np.max(np.abs(rep.singular_values[l] - fx[f"sv{l}"])) <= 1e-10 * fx[f"sv{l}"][0]
    np.testing.assert_allclose(rep.input_norm, fx["report"][3], rtol=1e-9)
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    assert np.max(np.abs(total.entries(pr) - fx["v_canonical"])) <= 1e-12 * scale
    v = tk.entries(pr)
    assert np.max(np.abs(v - fx["v_canonical"])) <= (10 * eps + 1e-12) * scale
    assert np.max(np.abs(v - fx["v_tucker"])) <= 1e-9 * scale
    nb = fx["v_brute"].size  # the reference's oracle_entry over the sources of both kernels
    assert np.max(np.abs(total.entries(pr[:nb]) - fx["v_brute"])) <= 1e-12 * scale
    # the same sum through the reference-shaped call: defected_sum(..., refs) with
    # DefectSpec-style (sites, charge, grid_offset, kernel) entries
    c = RF.CASES["mixed_kernels"]
    g0 = RF.geometry_parts("mixed_kernels")[0][2]
    ref_n = api.reference_for(g0, ctx)
    ref_y = api.reference_for(RF.geometry_parts("mixed_kernels")[1][2], ctx)
    defects = [(d[0], d[1], d[2], api.KernelSpec.yukawa(d[3][1]) if len(d) > 3 and d[3] else None)
               for d in c["defects"]]
    again = api.defected_sum(ref_n, c["cells"], c["n"], defects, cell_width=c["b"], refs=[ref_y])
    assert again.rank == total.rank
    np.testing.assert_array_equal(again.weights, total.weights)
    with pytest.raises(ValueError, match="no reference tensor"):
        api.defected_sum(ref_n, c["cells"], c["n"], defects, cell_width=c["b"])


def test_window_overflow_error_is_the_references(ctx):
    """A defect pushed outside the doubled grid: the reference throws WindowOverflowError
    (grid.hpp:87-98) naming the 1-based mode and the shift; the C ABI returns
    LATSUM_ERR_WINDOW_OVERFLOW with the same message."""
    if not RF.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    from paper_1411_1994_b200 import workload as W
    case = dict(cells=(4, 4, 4), n=16, b=1.0, family=0, lam=0.0, M=6, eps=1e-6,
                defects=[([(0, 0, 0)], -1.0, None), ([(1, 0, -1)], -1.0, (0.0, 40.0, 0.0))])
    r = RF.RefRun(case)
    try:
        with pytest.raises(RuntimeError) as ref_err:
            r.sum()
    finally:
        r.close()
    ref_msg = str(ref_err.value).split("): ", 1)[1]
    assert ref_msg.startswith("window overflow in mode 2: shift -40 pushes the length-64 window")
    g = W.from_lattice(case["cells"], case["n"], case["b"], M=case["M"], defects=case["defects"])
    with pytest.raises(api.WindowOverflowError) as err:
        api.lattice_sum(api.reference_for(g, ctx), g)
    assert ref_msg in str(err.value)
