"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE north star):
* directional vectors (unit side-matrix columns, stages 1-2): 1e-12 relative L-inf
  per column;
* truncated Tucker ranks: identical to the oracle's SVD ranks (a +-1 difference
  only at a flagged tie);
* reconstructed potentials: within 10*eps + 1e-12, normalised by max|oracle| over
  the probe set (commands.cpp:257-266), compared after reconstruction (sign freedom).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_1994_b200 import api
from paper_1411_1994_b200 import workload as W
from latsum_helpers import col_rel_linf, mini

pytestmark = pytest.mark.gpu

DIR_TOL = 1e-12


def _ref_pair(ctx, g):
    ref = api.reference_for(g, ctx)
    oref = O.reference(g)
    return ref, oref


# ----------------------------------------------------------------------------- stage 1

@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_stage1_reference_columns_match_oracle(ctx, cfg):
    g = W.baseline(cfg)
    ref, oref = _ref_pair(ctx, g)
    assert ref.rank == g.R == oref.weights.size
    assert ref.step_constant == oref.C0  # host sweep bit-identical
    t, a = ref.quadrature()
    assert np.array_equal(t, oref.nodes) and np.array_equal(a, oref.quad_weights)
    f = ref.factor(0)
    assert f.shape == (2 * g.N[0], g.R)
    assert col_rel_linf(f, oref.factors[0]) < DIR_TOL
    np.testing.assert_allclose(ref.weights, oref.weights, rtol=1e-13, atol=0)
    # identical modes share columns bitwise (test_reference.cpp:49-60)
    assert np.array_equal(ref.factor(2), f)


def test_stage1_zero_node_and_mirror(ctx):
    g = W.lattice_box(8, 2.0, [dict(cells=(2, 2, 2), step=(0.5, 0.5, 0.5))], M=6)
    ref = api.reference_for(g, ctx)
    f = ref.factor(0)
    n2 = f.shape[0]
    # t=0 column is constant before normalisation -> unit column 1/sqrt(2N)
    np.testing.assert_allclose(f[:, g.M], 1.0 / np.sqrt(n2), rtol=1e-14)
    np.testing.assert_allclose(f, f[::-1, :], rtol=1e-14, atol=0)  # mirror symmetry


# ----------------------------------------------------------------------------- stage 2

@pytest.mark.parametrize("kind", ["cubic", "vacancies", "yukawa", "hex", "mixed", "clusters"])
def test_stage2_side_matrices_match_oracle(ctx, kind):
    g = mini(kind)
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    F, w = O.side_matrices(oref, g)
    assert can.rank == g.canonical_rank
    for l in range(3):
        assert col_rel_linf(can.factor(l), F[l]) < DIR_TOL
    np.testing.assert_allclose(can.weights, w, rtol=1e-12, atol=0)


@pytest.mark.parametrize("cfg", [1, 2])
def test_stage2_full_config_side_matrices(ctx, cfg):
    g = W.baseline(cfg)
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    F, w = O.side_matrices(oref, g)
    for l in range(3):
        assert col_rel_linf(can.factor(l), F[l]) < DIR_TOL
    np.testing.assert_allclose(can.weights, w, rtol=1e-12, atol=0)


def test_stage2_assembled_equals_brute_force_oracle(ctx):
    g = mini("vacancies")
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    pr = O.probes(g.N, 300, 3)
    got = can.entries(pr)
    want = O.oracle_entries(oref, g, pr)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


def test_stage2_vacancy_is_base_minus_window(ctx):
    base = W.from_lattice((4, 4, 4), 16, M=8)
    vac = W.from_lattice((4, 4, 4), 16, M=8, defects=[([(0, 0, 0)], -1.0, None)])
    ref = api.reference_for(base, ctx)
    cb, cv = api.lattice_sum(ref, base), api.lattice_sum(ref, vac)
    assert cv.rank == 2 * ref.rank
    single = W.from_lattice((4, 4, 4), 16, M=8)
    single.sublattices = []
    single.defect_shifts = np.zeros((1, 3), np.int64)
    single.defect_charges = np.array([1.0])
    cw = api.lattice_sum(ref, single)
    pr = O.probes(base.N, 200, 5)
    lhs = cv.entries(pr)
    rhs = cb.entries(pr) - cw.entries(pr)
    assert np.max(np.abs(lhs - rhs)) / np.max(np.abs(lhs)) < 1e-12


def test_stage2_rectangular_clusters_assemble_at_reference_rank(ctx):
    """test_lattice_sum.cpp:273-305 through the C ABI: a 2 x 2 x 1 vacancy block is one
    assembled block (rank 2R), an L-shaped triple three windows (rank (1+3)R), and both
    match the brute-force oracle."""
    block = [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0)]
    ragged = [(2, 2, 0), (2, 3, 0), (3, 2, 0)]
    g0 = W.from_lattice((8, 8, 1), 8, M=8)
    ref = api.reference_for(g0, ctx)
    R = ref.rank
    c1 = api.lattice_sum(ref, W.from_lattice((8, 8, 1), 8, M=8, defects=[(block, -1.0, None)]))
    assert c1.rank == 2 * R
    c2 = api.lattice_sum(ref, W.from_lattice((8, 8, 1), 8, M=8, defects=[(ragged, -1.0, None)]))
    assert c2.rank == (1 + 3) * R
    g = W.from_lattice((8, 8, 1), 8, M=8, defects=[(block, -1.0, None), (ragged, -1.0, None)])
    both = api.lattice_sum(ref, g)
    assert both.rank == (1 + 1 + 3) * R
    oref = O.reference(g)
    pr = O.probes(g.N, 200, 12)
    want = O.oracle_entries(oref, g, pr)
    assert np.max(np.abs(both.entries(pr) - want) / np.abs(want)) < 1e-11
    F, w = O.side_matrices(oref, g)
    for l in range(3):
        assert col_rel_linf(both.factor(l), F[l]) < DIR_TOL
    np.testing.assert_allclose(both.weights, w, rtol=1e-12, atol=0)


def test_stage2_window_overflow_names_mode(ctx):
    g = W.from_lattice((4, 4, 4), 8, M=4)
    g.defect_shifts = np.array([[0, 40, 0]], np.int64)
    g.defect_charges = np.array([1.0])
    ref = api.reference_for(g, ctx)
    with pytest.raises(api.WindowOverflowError) as e:
        api.lattice_sum(ref, g)
    assert e.value.mode == 2


def test_stage2_empty_defects_is_identity(ctx):
    g = W.from_lattice((2, 2, 1), 8, M=6)
    ref = api.reference_for(g, ctx)
    a = api.lattice_sum(ref, g)
    b = api.lattice_sum(ref, W.from_lattice((2, 2, 1), 8, M=6, defects=[]))
    for l in range(3):
        assert np.array_equal(a.factor(l), b.factor(l))


# ----------------------------------------------------------------------------- stage 3

def _check_rhosvd(ctx, g, deflate="auto", probes=400):
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    F, w = O.side_matrices(oref, g)
    orc = O.rhosvd(F, w, eps=g.eps)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), deflate=deflate)
    for l in range(3):
        if rep.chosen_ranks[l] != orc.ranks[l]:
            assert orc.tie[l] or rep.tie_at_cutoff[l], (l, rep.chosen_ranks, orc.ranks)
            assert abs(rep.chosen_ranks[l] - orc.ranks[l]) <= 1
    assert t.ranks == rep.chosen_ranks
    # singular values relative to sigma_1 where resolved
    for l in range(3):
        s_gpu, s_orc = rep.singular_values[l], orc.sigma[l]
        assert s_gpu.size == s_orc.size
        assert np.max(np.abs(s_gpu - s_orc)) / s_orc[0] < 1e-10
    pr = O.probes(g.N, probes, 11)
    v_gpu = t.entries(pr)
    v_orc = O.projected_cp_entries(w, orc.Z, orc.P, pr)
    v_can = O.canonical_entries(F, w, pr)
    scale = np.max(np.abs(v_orc))
    assert np.max(np.abs(v_gpu - v_orc)) / scale <= 10 * g.eps + 1e-12
    assert np.max(np.abs(v_gpu - v_can)) / np.max(np.abs(v_can)) <= 10 * g.eps + 1e-12
    np.testing.assert_allclose(rep.weight_norm, orc.weight_norm, rtol=1e-12)
    np.testing.assert_allclose(rep.input_norm, orc.input_norm, rtol=1e-9)
    np.testing.assert_allclose(rep.bound_abs, orc.bound_abs, rtol=1e-3)
    return t, rep, orc


@pytest.mark.parametrize("kind", ["vacancies", "yukawa", "hex", "mixed", "clusters"])
def test_stage3_rhosvd_ranks_and_values(ctx, kind):
    _check_rhosvd(ctx, mini(kind))


def test_stage3_single_pass_vs_deflated(ctx):
    g = mini("mixed")
    t1, r1, orc = _check_rhosvd(ctx, g, deflate="always")
    assert all(r1.deflated)


def test_stage3_fixed_ranks_exact_low_rank(ctx):
    g = W.from_lattice((2, 2, 2), 8, M=3)  # canonical rank 7, merged 4 distinct terms
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.fixed_ranks(10, 10, 10))
    assert all(r <= 7 for r in rep.chosen_ranks)
    dense_t = t.to_dense()
    dense_c = can.to_dense()
    assert np.linalg.norm(dense_t - dense_c) / np.linalg.norm(dense_c) < 1e-12


def test_stage3_zero_tensor(ctx):
    g = W.from_lattice((2, 2, 2), 8, M=3)
    g.sublattices[0].charge = 0.0
    ref = api.reference_for(g, ctx)
    t, rep = api.rhosvd(api.lattice_sum(ref, g), api.TruncationSpec.fixed_ranks(2, 2, 2))
    assert rep.input_norm == 0.0 and rep.chosen_ranks == (1, 1, 1)
    assert np.all(t.to_dense() == 0.0)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [2, 3])
def test_stage3_full_config(ctx, cfg):
    _check_rhosvd(ctx, W.baseline(cfg), probes=300)


# ----------------------------------------------------------------------------- stage 4

def test_stage4_tucker_box_matches_entries(ctx):
    g = mini("hex")
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    lo, hi = (10, 20, 30), (90, 77, 130)
    box = t.to_dense(lo, hi)
    core = t.core
    U = [t.factor(l) for l in range(3)]
    rng = np.random.default_rng(1)
    pr = np.stack([rng.integers(lo[l], hi[l], 200) for l in range(3)], axis=1)
    want = O.tucker_entries(core, U, pr)
    got = box[pr[:, 0] - lo[0], pr[:, 1] - lo[1], pr[:, 2] - lo[2]]
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12
    np.testing.assert_allclose(t.entries(pr), want, rtol=0, atol=1e-12 * np.max(np.abs(want)))


def test_stage4_canonical_box_matches_oracle(ctx):
    g = W.baseline(1)
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    F, w = O.side_matrices(oref, g)
    plane = can.to_dense((0, 0, 256), (512, 512, 257))[:, :, 0]
    ii, jj = np.meshgrid(np.arange(0, 512, 7), np.arange(0, 512, 5), indexing="ij")
    pr = np.stack([ii.ravel(), jj.ravel(), np.full(ii.size, 256)], axis=1)
    want = O.canonical_entries(F, w, pr)
    got = plane[pr[:, 0], pr[:, 1]]
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12
    # axis lines against the brute-force windowed-sum oracle (lattice_sum.hpp:656-671)
    lines = []
    for l in range(3):
        p = np.full((512, 3), 256, np.int64)
        p[:, l] = np.arange(512)
        lines.append(p)
    pr = np.concatenate(lines)
    brute = O.oracle_entries(oref, g, pr)
    got = can.entries(pr)
    assert np.max(np.abs(got - brute)) / np.max(np.abs(brute)) < 1e-12


# ----------------------------------------------------------------------------- GEMM

@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(1, 1, 1), (37, 129, 17), (300, 260, 513), (64, 2000, 3000)])
def test_dgemm_dmma_matches_fp64_reference(ctx, ta, tb, shape):
    import torch
    M, N, K = shape
    g = torch.Generator().manual_seed(M * 7 + N + K)
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, generator=g)
    B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, generator=g)
    C = torch.randn((M, N), dtype=torch.float64, generator=g)
    want = 1.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.5 * C
    dA = A.T.contiguous().cuda()  # column-major storage == row-major transpose
    dB = B.T.contiguous().cuda()
    dC = C.T.contiguous().cuda()
    from paper_1411_1994_b200 import _lib
    lda = A.shape[0]
    ldb = B.shape[0]
    ctx.check(_lib.lib().latsum_dgemm_device(ctx.handle, ta, tb, M, N, K, 1.5, dA.data_ptr(), lda,
                                             dB.data_ptr(), ldb, -0.5, dC.data_ptr(), M))
    ctx.synchronize()
    got = dC.cpu().T
    err = (got - want).abs().max().item() / max(1.0, want.abs().max().item())
    assert err < 1e-13 * max(1, K) ** 0.5 * 10


@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("shape", [(1, 1, 1), (37, 129, 17), (128, 64, 32), (300, 1000, 366),
                                   (2048, 700, 384), (130, 70, 1000), (5, 3000, 2)])
def test_dgemm_ozaki_int8_matches_fp64(ctx, shape, tb):
    """The int8 tensor-core (tcgen05.mma.kind::i8) Ozaki GEMM C = A op(B) against an
    extended-precision product.  Error bound (ozaki_i8.cuh): K (2^-54 rounding of the
    lines + 6 * 2^-54 dropped digit pairs) max|A_i:| max|B_:j| + 2^-52 |C_ij| <=
    K 2^-51 max|A_i:| max|B_:j| + 2^-52 |C_ij|: FP64-GEMM accuracy relative to the
    row/column maxima.  Rows and columns span many binades and include zero lines."""
    import numpy as np
    import torch
    from paper_1411_1994_b200 import _lib
    M, N, K = shape
    rng = np.random.default_rng(M * 31 + N * 7 + K + tb)
    A = rng.standard_normal((M, K)) * np.exp2(rng.integers(-30, 30, size=(M, 1)))
    B = rng.standard_normal((K, N)) * np.exp2(rng.integers(-30, 30, size=(1, N)))
    A *= np.exp2(rng.integers(-6, 6, size=(M, K)))  # mixed exponents inside a row
    if M > 2:
        A[1, :] = 0.0
    if N > 3:
        B[:, 2] = 0.0
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F")).cuda()
    Bs = B.T if tb else B  # stored operand: op(Bs) = B
    dB = torch.from_numpy(np.asfortranarray(Bs).ravel(order="F")).cuda()
    dC = torch.full((M * N,), np.nan, dtype=torch.float64, device="cuda")
    ctx.check(_lib.lib().latsum_dgemm_ozaki_device(ctx.handle, tb, M, N, K, dA.data_ptr(), M,
                                                   dB.data_ptr(), Bs.shape[0], dC.data_ptr(), M))
    ctx.synchronize()
    got = dC.cpu().numpy().reshape((M, N), order="F")
    want = (A.astype(np.longdouble) @ B.astype(np.longdouble))
    amax = np.abs(A).max(axis=1, keepdims=True)
    bmax = np.abs(B).max(axis=0, keepdims=True)
    bound = (K * 2.0 ** -51) * amax * bmax + 2.0 ** -52 * np.abs(want).astype(np.float64)
    err = np.abs(got.astype(np.longdouble) - want).astype(np.float64)
    assert np.all(np.isfinite(got))
    assert np.all(err <= bound), float(np.max(err / np.maximum(bound, 1e-300)))
    # and against the DMMA GEMM (whose own error is within K 2^-53 (|A||B|)_ij <= bound)
    dmma = torch.empty_like(dC)
    ctx.check(_lib.lib().latsum_dgemm_device(ctx.handle, 0, tb, M, N, K, 1.0, dA.data_ptr(), M,
                                             dB.data_ptr(), Bs.shape[0], 0.0, dmma.data_ptr(), M))
    ctx.synchronize()
    ref = dmma.cpu().numpy().reshape((M, N), order="F")
    assert np.all(np.abs(got - ref) <= 2 * bound)


def test_dgemm_ozaki_long_k_is_split_and_accumulated(ctx):
    """K > 16384 (int32 accumulator headroom) runs as K-chunks accumulated into C in FP64
    (the beta path of the epilogue); checked against a long-double product."""
    import numpy as np
    import torch
    from paper_1411_1994_b200 import _lib
    M, N, K = 70, 130, 40000
    rng = np.random.default_rng(3)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    C0 = np.full((M, N), np.nan)
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F")).cuda()
    dB = torch.from_numpy(np.asfortranarray(B).ravel(order="F")).cuda()
    dC = torch.from_numpy(np.asfortranarray(C0).ravel(order="F").copy()).cuda()
    ctx.check(_lib.lib().latsum_dgemm_ozaki_device(ctx.handle, 0, M, N, K, dA.data_ptr(), M,
                                                   dB.data_ptr(), K, dC.data_ptr(), M))
    ctx.synchronize()
    got = dC.cpu().numpy().reshape((M, N), order="F")
    want = A.astype(np.longdouble) @ B.astype(np.longdouble)
    bound = (K * 2.0 ** -51) * np.abs(A).max(axis=1, keepdims=True) * np.abs(B).max(axis=0, keepdims=True)
    assert np.all(np.abs(got - want).astype(np.float64) <= bound + 2.0 ** -50 * np.abs(want).astype(np.float64))


# ----------------------------------------------------------------------------- full configs

@pytest.mark.slow
@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_config_against_oracle_fixture(ctx, cfg):
    """BASELINE configs at full size against the oracle fixtures of
    tests/golden/make_fullconfig.py (cfg5: factors-only RHOSVD, projected-CP values)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", f"fullcfg{cfg}.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    fx = np.load(path)
    g = W.baseline(cfg)
    ref = api.reference_for(g, ctx)
    assert ref.step_constant == float(fx["C0"])
    can = api.lattice_sum(ref, g)
    assert can.rank == int(fx["canonical_rank"])
    assert list(can.dict_cols) == list(fx["merged_columns"])
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), form_core=(cfg != 5))
    for l in range(3):
        fl = t.factor(l)
        assert np.all(np.isfinite(fl)), ("factor after rhosvd", l, int(np.sum(~np.isfinite(fl))),
                                         np.nonzero(~np.isfinite(fl).all(axis=1))[0][[0, -1]])
    ranks = list(fx["ranks"])
    for l in range(3):
        if rep.chosen_ranks[l] != ranks[l]:
            assert bool(fx["tie"][l]) or rep.tie_at_cutoff[l], (rep.chosen_ranks, ranks)
            assert abs(rep.chosen_ranks[l] - ranks[l]) <= 1
        s_orc = fx[f"sigma{l}"]
        s_gpu = rep.singular_values[l][:s_orc.size]
        assert rep.singular_values[l].size == int(fx["n_singular"][l])
        assert np.max(np.abs(s_gpu - s_orc)) / s_orc[0] < 1e-10
    pr = fx["probes"]
    v = t.entries(pr)
    want = fx["v_rhosvd"]
    assert np.max(np.abs(v - want)) / np.max(np.abs(want)) <= 10 * g.eps + 1e-12
    exact = can.entries(pr)
    np.testing.assert_allclose(exact, fx["v_canonical"], rtol=0,
                               atol=1e-12 * np.max(np.abs(fx["v_canonical"])))
    nb = fx["v_brute"].size
    assert np.max(np.abs(exact[:nb] - fx["v_brute"])) / np.max(np.abs(fx["v_brute"])) < 1e-12
    np.testing.assert_allclose(rep.weight_norm, float(fx["weight_norm"]), rtol=1e-12)
    np.testing.assert_allclose(rep.input_norm, float(fx["input_norm"]), rtol=1e-9)
    # singular values around the cut-off, per value (the rank rule reads this tail)
    for l in range(3):
        s_orc = fx[f"sigma{l}"]
        s_gpu = rep.singular_values[l][:s_orc.size]
        r = ranks[l]
        idx = np.arange(max(0, r - 64), min(s_orc.size, r + 64))
        idx = idx[s_orc[idx] >= 1e-2 * s_orc[r - 1]]  # values that weigh in the tail sum
        # per value in sigma^2 (what the tail sums add): 2e-6 relative (1e-6 in sigma), or a
        # shift of at most 3e-8 sigma_r^2 — the Gram's absolute resolution eps ||G2|| limits
        # values far under the cut (cfg5: sigma ~ 0.01 sigma_r to ~1e-5..1e-4 relative, and the
        # last digits there move from run to run with the concurrent streams' schedule: 5.6e-5
        # was seen once against 5e-5 allowed by 1e-8), the values at the cut are resolved to ~1e-9
        s2g, s2o, sr2 = s_gpu[idx] ** 2, s_orc[idx] ** 2, s_orc[r - 1] ** 2
        err = np.abs(s2g - s2o) - (2e-6 * s2o + 3e-8 * sr2)
        assert np.max(err) <= 0, (l, int(idx[np.argmax(err)]),
                                  float(np.max(np.abs(s_gpu[idx] - s_orc[idx]) / s_orc[idx])))
        near = np.abs(idx - r) <= 8  # the values deciding the rank: 1e-6 relative outright
        assert np.max(np.abs(s_gpu[idx[near]] - s_orc[idx[near]]) / s_orc[idx[near]]) < 1e-6
        # the tail the rank rule compares with eps ||sigma|| / 3 (rank_reduction.hpp:73-84)
        tail_g = np.sqrt(np.sum(rep.singular_values[l][r:] ** 2))
        tail_o = np.sqrt(np.sum(s_orc[r:] ** 2))
        assert abs(tail_g - tail_o) <= 1e-4 * tail_o, (l, tail_g, tail_o)
    # the benchmarked evaluation of the box, whole z-slices at the chunk boundaries
    _check_box_slices(ctx, t, g)


def _balanced_chunk(n, cap, align):
    """latsum_capi.cu balanced_chunk (the evaluation's z / y chunking)."""
    cap = max(1, cap)
    if n <= cap:
        return max(n, 1)
    parts = -(-n // cap)
    c = -(-n // parts)
    if align > 1 and c > align:
        c = min(cap, -(-c // align) * align)
    return max(1, min(c, cap))


def _box_slices(t, g, d0=None):
    """First and last z-slices of the evaluation box plus the two slices on each side of
    the first two z-chunk boundaries of the library's chunking (tucker_eval /
    cp_eval_grouped)."""
    lo, hi = g.eval_box()
    ni, nj, nk = (hi[l] - lo[l] for l in range(3))
    budget = 1 << 29
    if t.has_core:
        r0, r2 = t.ranks[0], t.ranks[2]
        njc = _balanced_chunk(nj, budget // max(r0 * r2, 1), 128)
        nkc = _balanced_chunk(nk, min(budget // max(r0 * njc, 1), 65535), 1)
    else:
        nkc = _balanced_chunk(nk, min(budget // max(nj * d0, 1), 65535), 1)
    ks = {0, nk - 1}
    for b in list(range(nkc, nk, nkc))[:2]:
        ks |= {b - 1, b}
    return sorted(ks), nkc


def _check_box_slices(ctx, t, g):
    """eval_box_device on the config's full evaluation box (the launch shape bench.py
    times: multi-chunk Ozaki slab chain, or cp_eval_grouped for factors-only tensors)
    against an FP64 evaluation on the host of the same tensor's core and factors
    (tucker.hpp:38-54 as a TTM chain) or projected form (V = sum_t w_t prod_l
    (U_l P_l)[i_l, c_l(t)]), whole z-slices, 1e-12 relative to the slices' max |V|."""
    import scipy.sparse as sp
    import torch
    lo, hi = g.eval_box()
    ni, nj, nk = (hi[l] - lo[l] for l in range(3))
    U = [t.factor(l)[lo[l]:hi[l]] for l in range(3)]
    if t.has_core:
        ks, nkc = _box_slices(t, g)
    else:
        P, tc, w = t.projected_form()
        D = [np.ascontiguousarray(U[l] @ P[l]) for l in range(3)]
        ks, nkc = _box_slices(t, g, D[0].shape[1])
    assert nkc < nk, "the box must span several z-chunks"
    ctx.trim_pool()  # room for the box next to the pool the context keeps
    torch.cuda.synchronize()
    out = torch.empty(ni * nj * nk, dtype=torch.float64, device="cuda")
    t.eval_box_device(lo, hi, out.data_ptr())
    ctx.synchronize()
    got = {k: out[k * ni * nj:(k + 1) * ni * nj].view(nj, ni).T.cpu().numpy() for k in ks}
    del out
    torch.cuda.empty_cache()
    if t.has_core:
        core = t.core
        r = t.ranks
        assert np.all(np.isfinite(core)), "core download"
        cm = core.reshape(r[0] * r[1], r[2], order="F")
        u2 = np.ascontiguousarray(U[2][ks].T)
        Q = np.empty((r[0] * r[1], len(ks)))
        step = 1 << 18  # row blocks: one BLAS call over 2.6e6 x 1266 returned NaN here once
        for a in range(0, cm.shape[0], step):
            Q[a:a + step] = cm[a:a + step] @ u2  # (r0 r1) x |ks|
        del core, cm
        assert all(np.all(np.isfinite(u)) for u in U), [int(np.sum(~np.isfinite(u))) for u in U]
        assert np.all(np.isfinite(Q)), int(np.sum(~np.isfinite(Q)))
        want = {k: U[0] @ Q[:, i].reshape(r[0], r[1], order="F") @ U[1].T for i, k in enumerate(ks)}
    else:
        want = {}
        for k in ks:
            M = sp.csr_matrix((w * D[2][k, tc[:, 2]], (tc[:, 0], tc[:, 1])),
                              shape=(D[0].shape[1], D[1].shape[1]))
            want[k] = np.asarray((M.T @ D[0].T).T) @ D[1].T
    for k in ks:
        assert np.all(np.isfinite(got[k])), (k, "device", int(np.sum(~np.isfinite(got[k]))))
        assert np.all(np.isfinite(want[k])), (k, "host", int(np.sum(~np.isfinite(want[k]))))
    scale = max(np.max(np.abs(v)) for v in want.values())
    for k in ks:
        err = np.max(np.abs(got[k] - want[k])) / scale
        assert err < 1e-12, (k, err)


@pytest.mark.parametrize("fixed_mode", [0, 1, 2])
def test_stage3_core_contracted_over_smallest_mode(ctx, fixed_mode):
    """Defects that share one coordinate make that mode's dictionary the smallest, so the
    core is contracted over mode 0, 1 or 2 (form_core); values must not depend on it."""
    sites = []
    for a in range(-2, 2):
        for b in range(-2, 2):
            s = [a, b]
            s.insert(fixed_mode, 0)
            sites.append(tuple(s))
    # one site short of the 4 x 4 x 1 product: a ragged cluster, one window per site
    # (a full product would be assembled at reference rank, lattice_sum.hpp:316-321)
    sites = sites[:-1]
    g = W.from_lattice((4, 4, 4), 16, M=6, defects=[(sites, -1.0, None)], eps=1e-7)
    assert g.n_defects == 15
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    assert int(np.argmin(can.dict_cols)) == fixed_mode
    F, w = O.side_matrices(oref, g)
    orc = O.rhosvd(F, w, eps=g.eps, with_norm=False)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    assert tuple(rep.chosen_ranks) == tuple(orc.ranks)
    core = O.project_core(w, orc.P)  # reference loop order, small sizes
    pr = O.probes(g.N, 300, 21)
    want = O.tucker_entries(core, orc.Z, pr)
    got = t.entries(pr)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-11


# ----------------------------------------------------------------------------- next rows

@pytest.mark.parametrize("kind", ["vacancies", "mixed"])
def test_gpu_bruteforce_verifier_matches_cpu_oracle(ctx, kind):
    """latsum_verify_entries = oracle_entry (lattice_sum.hpp:656-671) on the device."""
    g = mini(kind)
    ref, oref = _ref_pair(ctx, g)
    pr = O.probes(g.N, 200, 31)
    got = api.oracle_entries(ref, g, pr)
    want = O.oracle_entries(oref, g, pr)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-13
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    res = api.verify(t, ref, g, probes=300, seed=3, bound_abs=rep.bound_abs)
    assert res["ok"] and res["normalized"] <= 10 * g.eps + 1e-12


@pytest.mark.slow
def test_gpu_bruteforce_verifier_cfg5(ctx):
    """16.8M-source brute-force sum on the device vs the CPU oracle fixture."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "fullcfg5.npz")
    fx = np.load(path)
    g = W.baseline(5)
    ref = api.reference_for(g, ctx)
    nb = fx["v_brute"].size
    got = api.oracle_entries(ref, g, fx["probes"][:nb])
    assert np.max(np.abs(got - fx["v_brute"])) / np.max(np.abs(fx["v_brute"])) < 1e-12


@pytest.mark.parametrize("kind", ["vacancies", "hex"])
def test_canonical_to_tucker_matches_oracle(ctx, kind):
    """rank_reduction.hpp:280-306: rhosvd + ALS + shrink_core, against the oracle's
    restatement on full side matrices."""
    g = mini(kind)
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    F, w = O.side_matrices(oref, g)
    near = [False, False, False]
    core, Y, orc, sweeps = O.canonical_to_tucker(F, w, eps=g.eps, max_sweeps=3, near=near)
    t, rep, gsweeps = api.canonical_to_tucker(can, api.TruncationSpec.tol(g.eps), max_als_sweeps=3)
    for l in range(3):
        # identical ranks; +-1 only where the oracle's slice-drop decision was a tie
        # (the greedy drop loop interleaves the modes, so a tie in one mode moves the budget
        # every later decision sees: any flagged tie admits +-1)
        if rep.chosen_ranks[l] != core.shape[l]:
            assert any(near) and abs(rep.chosen_ranks[l] - core.shape[l]) <= 1, \
                (l, rep.chosen_ranks, core.shape, near)
        assert rep.chosen_ranks[l] <= orc.ranks[l]
    pr = O.probes(g.N, 300, 41)
    exact = O.canonical_entries(F, w, pr)
    got = t.entries(pr)
    want = O.tucker_entries(core, Y, pr)
    scale = np.max(np.abs(exact))
    assert np.max(np.abs(got - exact)) / scale <= 10 * g.eps
    assert np.max(np.abs(want - exact)) / scale <= 10 * g.eps
    assert gsweeps >= 1


def test_spectral_report_and_provenance_files(ctx, tmp_path):
    """cmd_sum's report and provenance sidecar (commands.cpp:56-72, report.cpp:28-73) for a
    clustered, truncated sum: the written values round-trip exactly (17 digits)."""
    g = mini("clusters")
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    rp, pp = tmp_path / "report.txt", tmp_path / "provenance.txt"
    api.write_spectral_report(str(rp), rep)
    api.write_provenance(str(pp), g, t, rep, seed=g.seed)
    lines = rp.read_text().splitlines()
    assert lines[0] == "# spectral report"
    assert lines[1] == "chosen_ranks %d %d %d" % rep.chosen_ranks
    assert float(lines[2].split()[1]) == rep.bound_abs
    for l in range(3):
        vals = np.array([float(x) for x in lines[8 + l].split()[1:]])
        assert np.array_equal(vals, rep.singular_values[l])
    prov = pp.read_text().splitlines()
    assert prov[:4] == ["# lattice sum provenance", f"seed {g.seed}", "grid %d %d %d" % g.N,
                        "cells 8 8 4"]
    assert prov[4:6] == ["format tucker", "ranks %d %d %d" % t.ranks]
    assert prov[6] == "summands 5"
    assert prov[7] == 'summand "assembled lattice sum" rank 21 sites 256'
    assert prov[8] == 'summand "vacancy cluster" rank 21 sites 4'
    assert prov[9] == 'summand "vacancy cluster" rank 63 sites 3'
    assert float(prov[-2].split()[1]) == rep.bound_abs


def test_tensor_files_match_reference_layout(ctx, tmp_path):
    """write_tensor / read_tensor (tensor_io.cpp:45-129): byte-identical to the oracle's
    restatement of the layout, round-trips, and rejects tampering (cli_pipeline.sh:87-90)."""
    g = W.from_lattice((2, 2, 2), 8, M=3, defects=[([(0, 0, 0)], -1.0, None)], eps=1e-6)
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    pt, pc = tmp_path / "t.tns", tmp_path / "c.tns"
    api.write_tensor(pt, t)
    api.write_tensor(pc, can)
    want_t = O.tensor_file_bytes("T", t.dims, t.ranks, [t.core] + [t.factor(l) for l in range(3)])
    assert pt.read_bytes() == want_t
    want_c = O.tensor_file_bytes("C", can.dims, [can.rank],
                                 [can.weights] + [can.factor(l) for l in range(3)])
    assert pc.read_bytes() == want_c
    t2 = api.read_tensor(pt, ctx)
    c2 = api.read_tensor(pc, ctx)
    pr = O.probes(g.N, 100, 2)
    np.testing.assert_array_equal(t2.entries(pr), t.entries(pr))
    np.testing.assert_allclose(c2.entries(pr), can.entries(pr), rtol=1e-13, atol=0)
    raw = bytearray(pt.read_bytes())
    raw[40] ^= 0x01
    pt.write_bytes(bytes(raw))
    with pytest.raises(IOError, match="checksum"):
        api.read_tensor(pt, ctx)


def _random_canonical(dims, rank, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(rank)
    F = []
    for l in range(3):
        f = rng.standard_normal((dims[l], rank))
        n = np.linalg.norm(f, axis=0)
        F.append(np.asfortranarray(f / n))
        w = w * n
    return w, F


@pytest.mark.parametrize("dims,rank", [((12, 12, 12), 3), ((20, 20, 20), 30), ((24, 24, 24), 12)])
def test_rhosvd_on_arbitrary_canonical_inputs(ctx, dims, rank):
    """test_rank_reduction.cpp:22-66 on the device: exact low rank, sigma vs an independent
    SVD (incl. the R > n case), error within the discarded-tail bound."""
    w, F = _random_canonical(dims, rank, 7 + rank)
    can = api.canonical_from_arrays(w, F, ctx)
    r = (3, 3, 3) if rank == 3 else (5, 5, 5)
    t, rep = api.rhosvd(can, api.TruncationSpec.fixed_ranks(*r))
    for l in range(3):
        s = np.linalg.svd(F[l], compute_uv=False)
        np.testing.assert_allclose(rep.singular_values[l][:s.size], s, rtol=1e-10, atol=1e-13 * s[0])
    dense = np.einsum("q,iq,jq,kq->ijk", w, F[0], F[1], F[2])
    approx = t.to_dense()
    err = np.linalg.norm(approx - dense)
    if rank == 3:
        assert err / np.linalg.norm(dense) < 1e-12
    assert err <= rep.bound_abs * (1 + 1e-12) + 1e-12 * np.linalg.norm(dense)


@pytest.mark.parametrize("kind", ["cubic", "vacancies", "yukawa"])
def test_canonical_box_eval_all_rank_buckets(ctx, kind):
    """Canonical to_dense on a box via the low-rank kernel (T <= 64) or the slab GEMMs."""
    g = mini(kind)
    ref, oref = _ref_pair(ctx, g)
    can = api.lattice_sum(ref, g)
    F, w = O.side_matrices(oref, g)
    lo, hi = (3, 0, 5), (g.N[0] - 2, g.N[1], 37)
    box = can.to_dense(lo, hi)
    rng = np.random.default_rng(4)
    pr = np.stack([rng.integers(lo[l], hi[l], 300) for l in range(3)], axis=1)
    want = O.canonical_entries(F, w, pr)
    got = box[pr[:, 0] - lo[0], pr[:, 1] - lo[1], pr[:, 2] - lo[2]]
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-12


@pytest.mark.parametrize("rank", [1, 2, 5, 17, 18, 23, 24, 25, 33, 47, 64])
def test_low_rank_canonical_eval_kernel_buckets(ctx, rank):
    """canonical.hpp:192-202 (to_dense) through k_cp_eval_small for every rank bucket
    (4 rows per thread up to 18 terms, 2 up to 24, then 1), on ragged boxes: row counts that
    are not multiples of the 128-thread row block, pair counts that are not multiples of the
    32-pair staging batch, and a pair range that wraps the j extent inside a batch."""
    dims = (700, 9, 13)
    w, F = _random_canonical(dims, rank, 100 + rank)
    can = api.canonical_from_arrays(w, F, ctx)
    for lo, hi in [((0, 0, 0), dims), ((3, 2, 1), (517, 9, 12)), ((100, 4, 0), (101, 5, 13))]:
        box = can.to_dense(lo, hi)
        want = np.einsum("q,iq,jq,kq->ijk", w, F[0][lo[0]:hi[0]], F[1][lo[1]:hi[1]],
                         F[2][lo[2]:hi[2]])
        assert box.shape == want.shape
        np.testing.assert_allclose(box, want, rtol=0, atol=1e-13 * np.max(np.abs(want)))


def test_assembly_term_merge_overlaps_and_joins(ctx):
    """The rank-1 term merge runs on a host thread after latsum_canonical_assemble returns:
    destroying the canonical at once must join it, and every consumer (merged-term count,
    entries, norm, RHOSVD) must see the finished merge; repeated assemblies agree exactly."""
    g = mini("vacancies")
    ref, oref = _ref_pair(ctx, g)
    for _ in range(3):  # create and drop without using the merged terms
        api.lattice_sum(ref, g)
    a = api.lattice_sum(ref, g)
    b = api.lattice_sum(ref, g)
    assert a.merged_terms == b.merged_terms > 0
    F, w = O.side_matrices(oref, g)
    pr = O.probes(g.N, 50, 3)
    np.testing.assert_array_equal(a.entries(pr), b.entries(pr))
    want = O.canonical_entries(F, w, pr)
    assert np.max(np.abs(a.entries(pr) - want)) / np.max(np.abs(want)) < 1e-12
    ta, ra = api.rhosvd(a, api.TruncationSpec.tol(g.eps))
    tb, rb = api.rhosvd(b, api.TruncationSpec.tol(g.eps))
    assert tuple(ra.chosen_ranks) == tuple(rb.chosen_ranks)
    assert abs(ra.input_norm - rb.input_norm) <= 1e-14 * ra.input_norm


@pytest.mark.parametrize("cfg", ["mini", 2])
def test_host_sink_streams_the_result(ctx, cfg):
    """latsum_ctx_set_host_sink: the core (chunk by chunk behind its contraction on cfg2's
    long-K path; whole on the small K-chunked path) and factors land in the host buffers,
    bit-identical to the explicit downloads."""
    import torch
    g = mini("vacancies") if cfg == "mini" else W.baseline(cfg)
    t0, _ = api.sum_to_tucker(g, g.eps, ctx)
    r = t0.ranks
    core = torch.zeros(int(np.prod(r)), dtype=torch.float64, pin_memory=True)
    fs = [torch.zeros(g.N[l] * r[l], dtype=torch.float64, pin_memory=True) for l in range(3)]
    ctx.set_host_sink(core.data_ptr(), core.numel(), [f.data_ptr() for f in fs],
                      [f.numel() for f in fs])
    try:
        t, _ = api.sum_to_tucker(g, g.eps, ctx)
    finally:
        ctx.set_host_sink(0, 0)
    assert t.sink_written and t.ranks == r
    assert np.array_equal(core.numpy(), t.core.ravel(order="F"))
    for l in range(3):
        assert np.array_equal(fs[l].numpy(), t.factor(l).ravel(order="F"))
    # too small a buffer: nothing streamed, the result stays on the device
    ctx.set_host_sink(core.data_ptr(), core.numel() - 1, [f.data_ptr() for f in fs],
                      [f.numel() for f in fs])
    try:
        t2, _ = api.sum_to_tucker(g, g.eps, ctx)
    finally:
        ctx.set_host_sink(0, 0)
    assert not t2.sink_written


_DMMA_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1411_1994_b200 import api, workload as W
g = W.baseline(int(sys.argv[2]))
ctx = api.Context(0)
ref = api.reference_for(g, ctx); can = api.lattice_sum(ref, g)
t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), form_core=False)
np.savez(sys.argv[3], ranks=np.array(rep.chosen_ranks), s0=rep.singular_values[0],
         s1=rep.singular_values[1], s2=rep.singular_values[2], tie=np.array(rep.tie_at_cutoff))
"""


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [4, 5])
def test_ozaki_stage3_matches_dmma_stage3(ctx, cfg, tmp_path):
    """The large configs' Grams, deflation projections and bases run on the Ozaki int8 GEMM;
    the same RHOSVD with every stage-3 GEMM on FP64 DMMA (LATSUM_GEMM_DMMA=1, a separate
    process: the switch is read once) gives the same ranks and the same spectrum at the
    cut (per value in sigma^2 units as in the fixture test) and tail sums to 1e-4."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for name, env in (("ozaki", {}), ("dmma", {"LATSUM_GEMM_DMMA": "1"})):
        f = tmp_path / f"{name}.npz"
        r = subprocess.run([sys.executable, "-c", _DMMA_SCRIPT, root, str(cfg), str(f)],
                           env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[name] = np.load(f)
    a, b = outs["ozaki"], outs["dmma"]
    assert list(a["ranks"]) == list(b["ranks"])
    for l in range(3):
        sa, sb = a[f"s{l}"], b[f"s{l}"]
        r = int(a["ranks"][l])
        idx = np.arange(max(0, r - 64), min(sa.size, r + 64))
        idx = idx[sb[idx] >= 1e-2 * sb[r - 1]]
        err = np.abs(sa[idx] ** 2 - sb[idx] ** 2) - (2e-6 * sb[idx] ** 2 + 3e-8 * sb[r - 1] ** 2)
        assert np.max(err) <= 0, (l, int(idx[np.argmax(err)]))
        ta, tb = np.sqrt(np.sum(sa[r:] ** 2)), np.sqrt(np.sum(sb[r:] ** 2))
        assert abs(ta - tb) <= 1e-4 * tb


def test_accumulation_orders_agree_and_sliding_is_the_references(ctx):
    """assembled_vector's orders (lattice_sum.hpp:101-144; test_lattice_sum.cpp:115-135): the
    sliding recursion (default, uniform strides) and the direct ascending sum agree to roundoff,
    both reproduce the reference's side matrices (tests/golden/refpin_*.npz, made with the
    reference's default sliding order), and a non-uniform list falls back to the direct sum."""
    import os
    from oracle import ref as RF
    for name in ("cubic", "clusters", "large"):
        g = RF.geometry(name)
        fx = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"refpin_{name}.npz"))
        got = {}
        try:
            for order in ("sliding", "ascending", "compensated"):
                ctx.set_accumulation(order)
                can = api.lattice_sum(api.reference_for(g, ctx), g)
                got[order] = ([can.factor(l) for l in range(3)], can.weights)
        finally:
            ctx.set_accumulation("sliding")
        cols = fx["F_cols"]
        for order, (F, w) in got.items():
            for l in range(3):
                assert col_rel_linf(F[l][:, cols], fx[f"F{l}"]) < 1e-12, (name, order, l)
            np.testing.assert_allclose(w, fx["weights"], rtol=1e-12)
        for l in range(3):
            d = np.max(np.abs(got["sliding"][0][l] - got["ascending"][0][l]))
            assert 0 < d < 1e-13, (name, l, d)  # different operation orders, same vectors
            assert np.array_equal(got["ascending"][0][l], got["compensated"][0][l])
    # non-uniform shift lists (BASELINE configs 2-5): both settings take the direct sum
    g = mini("vacancies")
    res = []
    try:
        for order in ("sliding", "ascending"):
            ctx.set_accumulation(order)
            res.append(api.lattice_sum(api.reference_for(g, ctx), g).factor(0))
    finally:
        ctx.set_accumulation("sliding")
    assert np.array_equal(res[0], res[1])
