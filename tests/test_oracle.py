"""Pins the CPU oracle (oracle/) against the reference's own known-answer and property
tests (/root/reference/proj/tests/unit/*.cpp) and the mpmath golden vectors in
tests/golden/.  No GPU needed."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_1994_b200 import workload as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def adaptive_simpson(f, a, b, tol=1e-13, depth=28):
    """test_helpers.hpp:75-94."""
    def rec(lo, hi, flo, fmid, fhi, whole, d):
        m = 0.5 * (lo + hi)
        lm, rm = 0.5 * (lo + m), 0.5 * (m + hi)
        flm, frm = f(lm), f(rm)
        left = (m - lo) / 6.0 * (flo + 4.0 * flm + fmid)
        right = (hi - m) / 6.0 * (fmid + 4.0 * frm + fhi)
        if d <= 0 or abs(left + right - whole) < 15.0 * tol:
            return left + right + (left + right - whole) / 15.0
        return rec(lo, m, flo, flm, fmid, left, d - 1) + rec(m, hi, fmid, frm, fhi, right, d - 1)
    m = 0.5 * (a + b)
    fa, fm, fb = f(a), f(m), f(b)
    return rec(a, b, fa, fm, fb, (b - a) / 6.0 * (fa + 4 * fm + fb), depth)


# ----------------------------------------------------------------------------- quadrature

@pytest.mark.parametrize("M", [2, 8, 19])
def test_rule_shape(M):
    """test_kernel_quadrature.cpp:23-38."""
    t, a = O.quadrature(0, 0.0, M, 2.5, 0.01, 1.0)
    assert t.size == 2 * M + 1 and t[M] == 0.0
    assert np.array_equal(t, -t[::-1]) and np.array_equal(a, a[::-1])
    assert np.all(a > 0)
    with pytest.raises(ValueError):
        O.quadrature(0, 0.0, 1, 1.0, 0.01, 1.0)


def test_yukawa_center_weight_vanishes():
    """test_kernel_quadrature.cpp:40-44."""
    t, a = O.quadrature(1, 1.0, 10, 2.5, 0.05, 5.0)
    assert a[10] == 0.0 and np.all(a >= 0)


def test_newton_rule_tracks_inverse_r():
    """test_kernel_quadrature.cpp:61-68: M=24, calibrated C0, |S(1) - 1| < 1e-5."""
    c0 = O.default_step_constant(0, 0.0, 24, 0.1, 10.0)
    t, a = O.quadrature(0, 0.0, 24, c0, 0.1, 10.0)
    for x in ([1.0, 0, 0], [0.6, 0.8, 0.0]):
        v = np.sum(a * np.exp(-(t * t)[:, None] * np.square(x)[None, :]).prod(axis=1))
        assert abs(v - 1.0) < 1e-5


def test_shell_error_decreases_with_M():
    """test_kernel_quadrature.cpp:70-86 (error ~ exp(-beta sqrt M), beta > 0.5)."""
    def err(M):
        c0 = O.default_step_constant(0, 0.0, M, 0.1, 10.0)
        t, a = O.quadrature(0, 0.0, M, c0, 0.1, 10.0)
        return O.lib().orc_shell_error(0, 0.0, O._ptr(t), O._ptr(a), t.size, 0.1, 10.0, 1000)
    e16, e32 = err(16), err(32)
    assert e32 < e16
    assert np.log(e16 / e32) / (np.sqrt(32) - 4.0) > 0.5


# ----------------------------------------------------------------------------- stage 1

def test_zero_node_column_is_cell_width():
    """test_reference.cpp:11-17 (grid cubic(2, 8), M=4, C0=2, shell [0.1, 2])."""
    t, _ = O.quadrature(0, 0.0, 4, 2.0, 0.1, 2.0)
    m = O.mode_integrals(t, 8, -1.0, 0.25, "literal")
    assert np.allclose(m[:, 4], 0.25, rtol=1e-15, atol=0)


@pytest.mark.parametrize("variant", ["literal", "hybrid"])
def test_mirrored_cells(variant):
    """test_reference.cpp:19-26."""
    t, _ = O.quadrature(0, 0.0, 6, 2.0, 0.1, 2.0)
    m = O.mode_integrals(t, 8, -1.0, 0.25, variant)
    np.testing.assert_allclose(m[:4], m[7:3:-1], rtol=1e-15, atol=0)


@pytest.mark.parametrize("variant", ["literal", "hybrid"])
def test_cell_integral_matches_adaptive_quadrature(variant):
    """test_reference.cpp:28-47: cell [0, 1] of [-2, 2] (h = 1)."""
    from math import erf, exp, pi, sqrt
    for tt in (0.35, 1.0, 3.7):
        m = O.mode_integrals(np.array([tt]), 4, -2.0, 1.0, variant)
        ref = adaptive_simpson(lambda x: exp(-tt * tt * x * x), 0.0, 1.0)
        assert abs(m[2, 0] - ref) <= 1e-12 * abs(ref)
        if tt == 1.0:
            assert abs(m[2, 0] - sqrt(pi) / 2 * erf(1.0)) <= 1e-15


def test_reference_shape_and_shared_modes():
    """test_reference.cpp:49-60: 2n rows, R = 2M+1, identical modes bitwise."""
    g = W.lattice_box(32, 4.0, [dict(cells=(2, 2, 2), step=(1, 1, 1))], M=10)
    ref = O.reference(g)
    assert ref.factors[0].shape == (64, 21)
    assert np.array_equal(ref.factors[0], ref.factors[1])
    assert np.array_equal(ref.factors[0], ref.factors[2])


def test_reference_entry_near_unit_radius():
    """test_reference.cpp:75-117: n=256, b=10, M=24, entry vs integrated 1/r, 1e-5."""
    g = W.Geometry(N=(256, 256, 256), box=(10.0, 10.0, 10.0), M=24)
    ref = O.reference(g)
    n2, h = 512, 10.0 / 256
    centers = -10.0 + (np.arange(n2) + 0.5) * h
    i1, i0 = int(np.argmin(np.abs(centers - 1.0))), int(np.argmin(np.abs(centers)))
    entry = np.sum(ref.weights * ref.factors[0][i1] * ref.factors[0][i0] * ref.factors[0][i0])
    gq = 12
    lo1, lo0 = -10.0 + i1 * h, -10.0 + i0 * h
    x = lo1 + (np.arange(gq) + 0.5) * h / gq
    y = lo0 + (np.arange(gq) + 0.5) * h / gq
    X, Y, Z = np.meshgrid(x, y, y, indexing="ij")
    integral = np.sum(1.0 / np.sqrt(X * X + Y * Y + Z * Z)) * (h / gq) ** 3
    assert abs(entry - integral) / abs(integral) < 1e-5


def test_golden_cell_integrals():
    """mpmath (50 digits) integrals of exp(-s x^2) over double-valued cells of the
    BASELINE grids (tests/golden/make_golden.py): hybrid within 1e-14 of the column
    maximum; the literal erf difference is reported, not gated."""
    data = json.load(open(os.path.join(GOLDEN, "cell_integrals.json")))
    worst_h, worst_l = 0.0, 0.0
    for rec in data["cells"]:
        s, lo, h = rec["s"], rec["lo"], rec["h"]
        node = np.array([np.sqrt(s)])
        hyb = O.mode_integrals(node, 1, lo, h, "hybrid")[0, 0]
        lit = O.mode_integrals(node, 1, lo, h, "literal")[0, 0]
        want = float(rec["value"])
        worst_h = max(worst_h, abs(hyb - want) / rec["colmax"])
        worst_l = max(worst_l, abs(lit - want) / rec["colmax"])
    assert worst_h < 1e-14, worst_h
    assert worst_l < 1e-9, worst_l


def test_golden_quadrature_and_step_constants():
    """Nodes/weights against 40-digit mpmath evaluation of quadrature.hpp:155-163 at the
    oracle's C0; C0 itself against the survey's independent probe (4 digits)."""
    data = json.load(open(os.path.join(GOLDEN, "quadrature.json")))
    for rec in data["configs"]:
        g = W.baseline(rec["cfg"])
        a, A = O.reference_shell(g.N, g.box)
        c0 = O.default_step_constant(g.family, g.lam, g.M, a, A)
        assert abs(c0 - rec["C0_probe"]) < 1e-4
        t, w = O.quadrature(g.family, g.lam, g.M, rec["C0"], a, A)
        np.testing.assert_allclose(t, np.array(rec["nodes"], float), rtol=4e-16, atol=0)
        gw = np.array(rec["weights"], float)
        # weights below 1e-20 of the largest sit at exp(-(lam/2)^2/t^2) arguments of
        # O(100), where 1 ulp in t moves the value by ~1e-14 relative: gate them absolutely
        np.testing.assert_allclose(w, gw, rtol=2e-15, atol=1e-20 * gw.max())


# ----------------------------------------------------------------------------- windows / geometry

def test_active_sets_and_snap():
    """test_grid_geometry.cpp:63-104."""
    assert list(W.default_active_set(2)) == [-1, 0]
    assert list(W.default_active_set(4)) == [-2, -1, 0, 1]
    assert list(W.default_active_set(1)) == [0]
    assert list(W.default_active_set(3)) == [-1, 0, 1]
    assert list(W.snap(np.array([1.4, -0.6, 0.0]), 1.0)) == [1, -1, 0]
    assert list(W.snap(np.array([0.5, -0.5, 0.0]), 1.0)) == [1, -1, 0]


def test_window_overflow_is_detected():
    """grid.hpp:104-114: a shift pushing the window out of the doubled grid."""
    col = np.ones(16)
    O.assembled_vector(col, 8, np.array([4]))
    with pytest.raises(OverflowError):
        O.assembled_vector(col, 8, np.array([5]))


# ----------------------------------------------------------------------------- stage 2

def _probe_err(F, w, ref, g, n=300, seed=2):
    pr = O.probes(g.N, n, seed)
    got = O.canonical_entries(F, w, pr)
    want = O.oracle_entries(ref, g, pr)
    return np.max(np.abs(got - want) / np.abs(want))


@pytest.mark.parametrize("L", [2, 4])
def test_assembled_sum_exact_against_brute_force(L):
    """test_lattice_sum.cpp:99-113."""
    g = W.from_lattice((L, L, L), 16, M=8)
    ref = O.reference(g)
    F, w = O.side_matrices(ref, g)
    assert w.size == ref.weights.size
    assert _probe_err(F, w, ref, g) < 1e-12


def test_sliding_and_ascending_orders_agree():
    """test_lattice_sum.cpp:115-128 (assembled_vector sliding vs ascending)."""
    g = W.from_lattice((8, 4, 2), 8, M=8)
    ref = O.reference(g)
    col = ref.factors[0][:, 3]
    N = 64
    asc = O.assembled_vector(col, N, np.arange(-4, 4) * 8)
    sl = np.zeros(N)
    O.lib().orc_assembled_vector_sliding(O._ptr(np.ascontiguousarray(col)), N, 8, 0, -4, 3,
                                         O._ptr(sl))
    assert np.max(np.abs(asc - sl)) / np.max(np.abs(asc)) < 1e-13


def test_vacancy_is_base_minus_window():
    """test_lattice_sum.cpp:198-232."""
    g = W.from_lattice((4, 4, 4), 16, M=8, defects=[([(0, 0, 0)], -1.0, None)])
    ref = O.reference(g)
    F, w = O.side_matrices(ref, g)
    assert w.size == 2 * ref.weights.size
    assert _probe_err(F, w, ref, g, 400, 6) < 1e-12


BLOCK_2x2 = [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0)]
RAGGED_L = [(2, 2, 0), (2, 3, 0), (3, 2, 0)]


def test_product_structure_detection():
    """lattice_sum.hpp:278-294: full Cartesian products only (every combination once)."""
    assert W.product_structure(BLOCK_2x2) == [[0, 1], [0, 1], [0]]
    assert W.product_structure(RAGGED_L) is None
    assert W.product_structure([(0, 0, 0), (0, 0, 0)]) is None  # repeated site
    assert W.product_structure([(5, -1, 2)]) == [[5], [-1], [2]]
    assert W.product_structure([(a, b, c) for c in (1, 3) for b in (0, 2, 4) for a in (-1, 7)]) \
        == [[-1, 7], [0, 2, 4], [1, 3]]


def test_rectangular_clusters_assemble_at_reference_rank():
    """test_lattice_sum.cpp:273-305: the 2 x 2 x 1 vacancy block is assembled (rank 2R, not
    4 windows), the L-shaped triple has no product structure (rank (1+3)R), and both
    forms agree with the brute-force oracle."""
    R = 17
    g1 = W.from_lattice((8, 8, 1), 8, M=8, defects=[(BLOCK_2x2, -1.0, None)])
    assert g1.canonical_rank == 2 * R
    g2 = W.from_lattice((8, 8, 1), 8, M=8, defects=[(RAGGED_L, -1.0, None)])
    assert g2.canonical_rank == (1 + 3) * R
    g = W.from_lattice((8, 8, 1), 8, M=8, defects=[(BLOCK_2x2, -1.0, None),
                                                    (RAGGED_L, -1.0, None)])
    ref = O.reference(g)
    F, w = O.side_matrices(ref, g)
    assert w.size == (1 + 1 + 3) * R == g.canonical_rank
    assert _probe_err(F, w, ref, g, 200, 12) < 1e-11
    # the assembled cluster block equals the sum of its four windows
    gs = W.from_lattice((8, 8, 1), 8, M=8)
    gs.defect_shifts, gs.defect_charges = g.defect_shifts[:4], g.defect_charges[:4]
    Fs, ws = O.side_matrices(ref, gs)
    pr = O.probes(g.N, 300, 5)
    blk = O.canonical_entries([f[:, R:2 * R] for f in F], w[R:2 * R], pr)
    four = O.canonical_entries([f[:, R:] for f in Fs], ws[R:], pr)
    assert np.max(np.abs(blk - four)) <= 1e-12 * np.max(np.abs(four))


def test_offgrid_defect_snaps_to_grid():
    """test_lattice_sum.cpp:308-330 (off-grid impurity at grid_offset (3, -2, 0))."""
    g = W.from_lattice((4, 4, 1), 8, M=8, defects=[([(0, 0, 0)], 0.5, (3.0, -2.0, 0.0))])
    assert g.defect_shifts.tolist() == [[3, -2, 0]]
    ref = O.reference(g)
    F, w = O.side_matrices(ref, g)
    assert _probe_err(F, w, ref, g, 200, 14) < 1e-11


def test_hexagonal_union_matches_brute_force():
    """test_lattice_sum.cpp:396-424."""
    g = W.from_lattice((4, 4, 1), 8, M=8, sublattices=[((2, 2, 1), (0, 0, 0)),
                                                       ((2, 2, 1), (0.5, 0.5, 0.0))],
                       parent_cells=(4, 4, 1))
    ref = O.reference(g)
    F, w = O.side_matrices(ref, g)
    assert w.size == 2 * ref.weights.size
    assert _probe_err(F, w, ref, g, 200, 16) < 1e-12


def test_translation_covariance():
    """test_lattice_sum.cpp:140-158."""
    g1 = W.from_lattice((6, 1, 1), 8, M=8, active=[[-2, -1, 0, 1], [], []])
    g2 = W.from_lattice((6, 1, 1), 8, M=8, active=[[-1, 0, 1, 2], [], []])
    ref = O.reference(g1)
    F1, w1 = O.side_matrices(ref, g1)
    F2, w2 = O.side_matrices(ref, g2)
    n = 8
    a = F2[0][n:] * w2[None, :]
    b = F1[0][:-n] * w1[None, :]
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14 * np.abs(b).max())


# ----------------------------------------------------------------------------- stage 3

def _random_canonical(dims, rank, seed):
    rng = np.random.default_rng(seed)
    F = []
    w = rng.standard_normal(rank)
    for l in range(3):
        f = rng.standard_normal((dims[l], rank))
        nrm = np.linalg.norm(f, axis=0)
        F.append(np.asfortranarray(f / nrm))
        w = w * nrm
    return F, w


def _dense_canonical(F, w):
    return np.einsum("q,iq,jq,kq->ijk", w, F[0], F[1], F[2])


def _dense_tucker(core, Z):
    return np.einsum("abc,ia,jb,kc->ijk", core, Z[0], Z[1], Z[2])


def test_rhosvd_exact_low_rank():
    """test_rank_reduction.cpp:22-28."""
    F, w = _random_canonical((12, 12, 12), 3, 3)
    r = O.rhosvd(F, w, ranks=(3, 3, 3))
    core = O.project_core(w, r.P)
    A = _dense_canonical(F, w)
    assert np.linalg.norm(_dense_tucker(core, r.Z) - A) / np.linalg.norm(A) < 1e-12
    assert r.ranks == (3, 3, 3)


def test_rhosvd_error_within_bound():
    """test_rank_reduction.cpp:43-51."""
    for trial in range(5):
        F, w = _random_canonical((24, 24, 24), 12, 100 + trial)
        r = O.rhosvd(F, w, ranks=(5, 5, 5))
        err = np.linalg.norm(_dense_tucker(O.project_core(w, r.P), r.Z) - _dense_canonical(F, w))
        assert err <= r.bound_abs * (1 + 1e-12)


def test_rhosvd_singular_values_match_independent_svd():
    """test_rank_reduction.cpp:53-66 (R > n exercises the wide case)."""
    F, w = _random_canonical((20, 20, 20), 30, 55)
    r = O.rhosvd(F, w, ranks=(4, 4, 4))
    for l in range(3):
        s = np.linalg.svd(F[l], compute_uv=False)
        np.testing.assert_allclose(r.sigma[l], s, rtol=1e-10)


def test_rhosvd_norms_and_stability():
    F, w = _random_canonical((10, 10, 10), 6, 9)
    r = O.rhosvd(F, w, ranks=(3, 3, 3))
    np.testing.assert_allclose(r.input_norm, np.linalg.norm(_dense_canonical(F, w)), rtol=1e-12)
    np.testing.assert_allclose(r.weight_norm, np.linalg.norm(w), rtol=1e-15)


def test_merged_svd_equals_full_svd_on_lattice_sum():
    """The column-merged SVD the oracle uses has the reference's singular values."""
    g = W.from_lattice((4, 4, 4), 8, M=6, defects=[([(0, 0, 0), (1, 0, 0)], -1.0, None)])
    ref = O.reference(g)
    F, w = O.side_matrices(ref, g)
    r = O.rhosvd(F, w, eps=1e-6)
    for l in range(3):
        s = np.linalg.svd(F[l], compute_uv=False)
        n = r.sigma[l].size
        np.testing.assert_allclose(r.sigma[l][:n], s[:n], rtol=0, atol=1e-13 * s[0])


def test_rank_for_tolerance_rule():
    """rank_reduction.hpp:73-84 on a hand-made spectrum."""
    sv = np.array([1.0, 0.1, 0.01, 1e-3, 1e-4])
    nrm = np.linalg.norm(sv)
    # eps chosen so that tail(3) = ||[1e-3, 1e-4]|| is just inside the target
    eps = 3 * np.linalg.norm(sv[3:]) / nrm * 1.0001
    assert O.rank_for_tolerance(sv, eps) == 3
    assert O.rank_for_tolerance(sv, eps * 0.999) == 4
    assert O.rank_for_tolerance(sv, 0.9999) == 1
