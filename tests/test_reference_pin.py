"""Pinning the oracle to the REFERENCE ITSELF (no GPU).

oracle/_ref is the reference's own headers and unit tests compiled where they lie under
/root/reference against the stand-ins for its two absent third-party headers (oracle/shim).
tests/golden/refpin_*.npz hold its outputs on geometries its API can express
(tests/golden/make_refpin.py).  Here:

* the reference's own unit-test suite passes on that build (the stand-ins are faithful);
* the fixtures equal what the live reference library produces now (when it is present);
* the CPU restatement (oracle.py / latsum_oracle.cpp) reproduces the reference's outputs:
  C0, nodes and weights bit for bit, side matrices to 1e-13, identical RHOSVD ranks, singular
  values to 1e-12 sigma_1, Tucker entries to 1e-11, the brute-force sum to 1e-13.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))

from oracle import oracle as O  # noqa: E402
from oracle import ref as RF  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = RF.single_kernel_cases()
HAVE_REFERENCE = os.path.isdir(os.path.join(RF.REFERENCE_ROOT, "include", "latsum"))


def fixture(name):
    return np.load(os.path.join(GOLD, f"refpin_{name}.npz"))


@pytest.fixture(scope="module")
def ref_built():
    if HAVE_REFERENCE:
        assert RF.build()
    elif not RF.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return True


def test_reference_unit_tests_pass_on_the_standins(ref_built):
    """The reference's tests/unit suite (89 cases; test_io_config needs nlohmann json) on the
    reference compiled against oracle/shim."""
    line = RF.run_unit_tests()
    assert "| 0 failed; assertions:" in line and line.endswith("rc=0"), line
    n_cases = int(line.split("test cases:")[1].split("|")[0])
    assert n_cases >= 89, line


def test_reference_acceptance_program_passes(ref_built):
    """The reference's tests/acceptance/acceptance_main.cpp (9 criteria: reference accuracy,
    assembled exactness, Tucker sums, RHOSVD / ALS bounds, defect algebra, O(L) scaling through its
    own cmd_bench, Galerkin, quadrature slope) on the reference compiled against oracle/shim."""
    import subprocess
    out = subprocess.run([os.path.join(os.path.dirname(RF.SO), "ref_acceptance")],
                         capture_output=True, text=True, timeout=900)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("[")]
    assert len(lines) == 9, out.stdout
    # criterion 7 fits wall-clock scaling exponents (its own gate: exponent <= 1.3 within 300 s):
    # the only one that may depend on the load of the host the suite runs on
    failed = [ln for ln in lines if not ln.startswith("[PASS]")]
    assert all("criterion 7" in ln for ln in failed), out.stdout


@pytest.mark.parametrize("name", ["clusters", "union", "vacancies"])
def test_reference_cmd_sum_and_cmd_verify(ref_built, name, tmp_path):
    """The reference's own `latsum sum` and `latsum verify` (src/commands.cpp:108-177, 200-284)
    through oracle/_ref: the truncated sum it writes passes its own 500-probe check against the
    recorded bound, and its ranks are the library-level canonical_to_tucker ranks of the fixture
    (the union case without its defects: cmd_sum's sublattice route takes none)."""
    fx = fixture(name)
    r = RF.RefRun(name)
    try:
        tp, pp = tmp_path / "t.tns", tmp_path / "p.txt"
        log = r.cmd_sum(eps=RF.CASES[name]["eps"], max_als_sweeps=int(fx["c2t_sweeps"]), seed=5,
                        tensor_path=tp, provenance_path=pp, report_path=tmp_path / "r.txt")
        assert "wrote tensor" in log and "wrote provenance" in log
        ranks = r.tucker()["ranks"]
        if name != "union":
            assert ranks == tuple(int(x) for x in fx["c2t_ranks"])
        ok, vlog, err = r.cmd_verify(tp, pp, probes=500, seed=5)
        assert ok and vlog.rstrip().endswith("verify: ok"), (vlog, err)
        raw = bytearray(tp.read_bytes())
        raw[len(raw) // 2] ^= 0x04
        tp.write_bytes(bytes(raw))
        ok, vlog, err = r.cmd_verify(tp, pp, probes=10, seed=5)
        assert not ok and "checksum" in err
    finally:
        r.close()


@pytest.mark.parametrize("name", [c for c in RF.CASES if c != "large"])
def test_fixtures_equal_the_live_reference(ref_built, name):
    import make_refpin
    live = make_refpin.derive(name)
    fx = fixture(name)
    assert set(live) == set(fx.files)
    for k, v in live.items():
        assert np.array_equal(np.asarray(v), fx[k]), k


def test_reference_helpers_match_the_port(ref_built):
    """assembled_vector's three accumulation orders and rank_for_tolerance, reference vs port."""
    rng = np.random.default_rng(3)
    ref_col = rng.standard_normal(128)
    ks = np.array([-2, -1, 0, 1])
    want = O.assembled_vector(ref_col, 64, ks * 16 + 3)
    for acc in (0, 1, 2):
        got = RF.assembled_vector(ref_col, ks, 16, 3, 64, acc)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-14)
    sv = np.sort(np.abs(rng.standard_normal(40)) * 10.0 ** rng.uniform(-9, 0, 40))[::-1].copy()
    for eps in (1e-2, 1e-4, 1e-6, 1e-8):
        assert RF.rank_for_tolerance(sv, eps) == O.rank_for_tolerance(sv, eps)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_baseline_quadrature_is_the_references(ref_built, cfg):
    """C0 sweep, nodes and weights of the five BASELINE shells: reference == port, bit for bit."""
    from paper_1411_1994_b200 import workload as W
    g = W.baseline(cfg)
    a, A = O.reference_shell(g.N, g.box)
    c0, t, w = RF.quadrature(g.family, g.lam, g.M, 0.0, a, A)
    assert c0 == O.default_step_constant(g.family, g.lam, g.M, a, A)
    nodes, qw = O.quadrature(g.family, g.lam, g.M, c0, a, A)
    assert np.array_equal(t, nodes) and np.array_equal(w, qw)


@pytest.mark.parametrize("name", CASES)
def test_port_reproduces_the_reference(name):
    fx = fixture(name)
    g = RF.geometry(name)
    assert tuple(g.N) == tuple(int(x) for x in fx["N"])
    # ---- stage 1
    lit = O.reference(g, variant="literal")
    hyb = O.reference(g)
    assert lit.C0 == float(fx["C0"])
    assert np.array_equal(lit.nodes, fx["nodes"]) and np.array_equal(lit.quad_weights, fx["quad_weights"])
    for l in range(3):
        assert np.max(np.abs(lit.factors[l] - fx[f"ref_factor{l}"])) < 1e-15   # the literal formula
        assert np.max(np.abs(hyb.factors[l] - fx[f"ref_factor{l}"])) < 1e-13   # hybrid cells (DESIGN 3)
    np.testing.assert_allclose(hyb.weights, fx["ref_weights"], rtol=1e-13)
    # ---- stage 2: same term order, same columns, same weights, same provenance
    F, w = O.side_matrices(hyb, g)
    assert w.size == fx["weights"].size == g.canonical_rank
    cols = fx["F_cols"]
    for l in range(3):
        assert np.max(np.abs(F[l][:, cols] - fx[f"F{l}"])) < 1e-13
    np.testing.assert_allclose(w, fx["weights"], rtol=1e-12, atol=1e-15 * np.abs(w).max())
    assert [s[0] for s in g.summands()] == [str(x) for x in fx["summand_labels"]]
    assert [s[1] for s in g.summands()] == fx["summand_ranks"].tolist()
    assert [s[2] for s in g.summands()] == fx["summand_sites"].tolist()
    # ---- stage 3
    orc = O.rhosvd(F, w, eps=g.eps)
    assert tuple(orc.ranks) == tuple(int(x) for x in fx["ranks"])
    assert tuple(orc.tie) == tuple(bool(x) for x in fx["ties"])
    for l in range(3):
        sv = fx[f"sv{l}"]
        assert orc.sigma[l].size == sv.size
        assert np.max(np.abs(orc.sigma[l] - sv)) <= 1e-12 * sv[0]
    bound_abs, bound_rel, weight_norm, input_norm, stab, stab_ok = fx["report"]
    np.testing.assert_allclose(orc.weight_norm, weight_norm, rtol=1e-13)
    np.testing.assert_allclose(orc.input_norm, input_norm, rtol=1e-12)
    np.testing.assert_allclose(orc.stability_constant, stab, rtol=1e-11)
    # the tail sums lose digits to the values they discard (~1e-16 sigma_1 noise each)
    noise = 1e-13 * weight_norm * fx["sv0"][0]
    np.testing.assert_allclose(orc.bound_abs, bound_abs, rtol=1e-6, atol=noise)
    np.testing.assert_allclose(orc.bound_rel, bound_rel, rtol=1e-6, atol=noise * 10)
    # ---- stage 4
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    assert np.max(np.abs(O.canonical_entries(F, w, pr) - fx["v_canonical"])) <= 1e-13 * scale
    assert np.max(np.abs(O.projected_cp_entries(w, orc.Z, orc.P, pr) - fx["v_tucker"])) <= 1e-11 * scale
    nb = fx["v_brute"].size
    assert np.max(np.abs(O.oracle_entries(hyb, g, pr[:nb]) - fx["v_brute"])) <= 1e-13 * scale
    # the reference's own truncation error stays within its tolerance (commands.cpp:257-266)
    assert np.max(np.abs(fx["v_tucker"] - fx["v_canonical"])) <= 10 * g.eps * scale


@pytest.mark.parametrize("name", ["vacancies", "yukawa", "union", "clusters"])
def test_port_canonical_to_tucker_matches_the_reference(name):
    """rank_reduction.hpp:280-306 with 3 ALS sweeps: the port's ranks are the reference's (+-1
    only where the port's own slice-drop decision was a flagged tie) and both stay within
    tolerance of the exact sum."""
    fx = fixture(name)
    g = RF.geometry(name)
    F, w = O.side_matrices(O.reference(g), g)
    near = [False, False, False]
    core, Y, orc, sweeps = O.canonical_to_tucker(F, w, eps=g.eps, max_sweeps=int(fx["c2t_sweeps"]), near=near)
    want = tuple(int(x) for x in fx["c2t_ranks"])
    for l in range(3):
        if core.shape[l] != want[l]:
            assert any(near) and abs(core.shape[l] - want[l]) <= 1, (core.shape, want, near)
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    # shrink_core spends the whole Frobenius budget eps ||A||, so pointwise errors sit a little
    # above rhosvd's; the port and the reference land on the same values
    got = O.tucker_entries(core, Y, pr)
    assert np.max(np.abs(got - fx["v_canonical"])) <= 30 * g.eps * scale
    assert np.max(np.abs(fx["v_c2t"] - fx["v_canonical"])) <= 30 * g.eps * scale
    if core.shape == want:
        assert np.max(np.abs(got - fx["v_c2t"])) <= 3 * g.eps * scale


class _Rank:  # stands in for a device CanonicalTensor / TuckerTensor (format + ranks only)
    def __init__(self, rank=None, ranks=None):
        if rank is not None:
            self.rank = rank
        else:
            self.ranks = ranks


@pytest.mark.parametrize("name", ["clusters", "union", "cubic"])
def test_report_writers_match_the_references(ref_built, name):
    """latsum_format_spectral_report / latsum_format_provenance (host-only C ABI) against the
    reference's own write_spectral_report / write_provenance (src/report.cpp:28-73, compiled into
    oracle/_ref) on the same numbers: identical text."""
    from paper_1411_1994_b200 import api
    g = RF.geometry(name)
    r = RF.RefRun(name)
    try:
        r.sum()
        red = r.reduce("rhosvd", eps=g.eps)
        want_report = r.spectral_report_text()
        want_prov_t = r.provenance_text(2 ** 64 - 3, True, "note x")
        want_prov_c = r.provenance_text(7, False)
        n_terms = r.canonical()[1].size
    finally:
        r.close()
    rep = api.SpectralReport(
        singular_values=red["sv"], chosen_ranks=red["ranks"], bound_abs=red["bound_abs"],
        bound_rel=red["bound_rel"], weight_norm=red["weight_norm"], input_norm=red["input_norm"],
        stability_constant=red["stability_constant"], stability_ok=red["stability_ok"],
        tie_at_cutoff=red["ties"], cutoff_margin=(0.0, 0.0, 0.0), deflated=(False,) * 3,
        gram_rows=(False,) * 3, gram_size=(0, 0, 0), ms={})
    assert api.format_spectral_report(rep) == want_report
    assert api.format_provenance(g, _Rank(ranks=red["ranks"]), rep, seed=2 ** 64 - 3,
                                 extra_lines=["note x"]) == want_prov_t
    assert api.format_provenance(g, _Rank(rank=n_terms), seed=7) == want_prov_c
    # and the oracle's restatements, which the GPU-side tests use
    assert O.spectral_report_text(red["ranks"], red["bound_abs"], red["bound_rel"], red["weight_norm"],
                                  red["input_norm"], red["stability_constant"], red["stability_ok"],
                                  red["ties"], red["sv"]) == want_report


def test_tensor_file_layout_is_the_references(ref_built, tmp_path):
    """write_tensor / read_tensor (src/tensor_io.cpp, compiled into oracle/_ref): the oracle's
    restatement of the layout (which the product's writer equals byte for byte,
    test_tensor_files_match_reference_layout) produces the reference's bytes; the reference reads
    them back and rejects a flipped bit."""
    r = RF.RefRun("cubic")
    try:
        r.sum()
        F, w = r.canonical()
        red = r.reduce("rhosvd", eps=RF.CASES["cubic"]["eps"])
        pc, pt = tmp_path / "c.tns", tmp_path / "t.tns"
        r.write_tensor("canonical", pc)
        r.write_tensor("tucker", pt)
        pr = O.probes((64, 64, 64), 50, 5)
        want_c, want_t = r.entries("canonical", pr), r.entries("tucker", pr)
    finally:
        r.close()
    assert pc.read_bytes() == O.tensor_file_bytes("C", (64, 64, 64), [w.size], [w] + F)
    assert pt.read_bytes() == O.tensor_file_bytes("T", (64, 64, 64), red["ranks"], [red["core"]] + red["U"])
    kind, dims, got = RF.read_tensor_entries(pt, pr)
    assert kind == "tucker" and dims == (64, 64, 64) and np.array_equal(got, want_t)
    kind, dims, got = RF.read_tensor_entries(pc, pr)
    assert kind == "canonical" and np.array_equal(got, want_c)
    raw = bytearray(pt.read_bytes())
    raw[40] ^= 0x01
    pt.write_bytes(bytes(raw))
    with pytest.raises(IOError):
        RF.read_tensor_entries(pt, pr)


def test_port_reproduces_per_defect_kernels():
    """DefectSpec.kernel (geometry.hpp:26, lattice_sum.hpp:301-303): clusters carrying their own
    kernel are assembled against that kernel's reference tensor and concatenated in DefectSpec
    order (add_concat, canonical.hpp:94-110).  The port's per-part side matrices, concatenated,
    are the reference's."""
    fx = fixture("mixed_kernels")
    Fs, ws = [[], [], []], []
    for fam, lam, g in RF.geometry_parts("mixed_kernels"):
        F, w = O.side_matrices(O.reference(g), g)
        for l in range(3):
            Fs[l].append(F[l])
        ws.append(w)
    F = [np.hstack(x) for x in Fs]
    w = np.concatenate(ws)
    assert w.size == fx["weights"].size == 105
    for l in range(3):
        assert np.max(np.abs(F[l][:, fx["F_cols"]] - fx[f"F{l}"])) < 1e-13
    np.testing.assert_allclose(w, fx["weights"], rtol=1e-12)
    orc = O.rhosvd(F, w, eps=RF.CASES["mixed_kernels"]["eps"])
    assert tuple(orc.ranks) == tuple(int(x) for x in fx["ranks"])
    pr = fx["probes"]
    scale = np.max(np.abs(fx["v_canonical"]))
    assert np.max(np.abs(O.canonical_entries(F, w, pr) - fx["v_canonical"])) <= 1e-13 * scale
    assert np.max(np.abs(fx["v_brute"] - fx["v_canonical"][:fx["v_brute"].size])) <= 1e-12 * scale
