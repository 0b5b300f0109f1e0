"""The library's row-sharded RHOSVD executed for real: two ranks as two contexts
on one device, driven from two host threads, exchanging partial Grams / projections /
eigensolves / Z row blocks / core shares through host collectives (latsum_ctx_init_host_comm;
the NCCL path calls the same collectives).  No kernel waits on another rank's kernel: every
exchange happens on the host between stream synchronisations."""
import os
import threading

import numpy as np
import pytest

from oracle import oracle as O
from paper_1411_1994_b200 import api
from paper_1411_1994_b200 import workload as W

pytestmark = pytest.mark.gpu


def _run_ranks(g, nranks, form_core=True, core_slabs=False, box=None):
    coll = api.ThreadCollective(nranks)
    out, errs = [None] * nranks, []

    def rank_main(q):
        try:
            ctx = api.Context(0)
            api.init_host_comm(ctx, q, nranks, coll)
            ref = api.reference_for(g, ctx)
            can = api.lattice_sum(ref, g)
            t, rep = api.rhosvd(can, api.TruncationSpec.tol(g.eps), form_core=form_core,
                                core_slabs=core_slabs)
            vals = None
            if box is not None:  # the ranks evaluate together (partial boxes + all-reduce)
                vals = t.to_dense(*box)
            out[q] = (ctx, can, t, rep) if box is None else (ctx, can, t, rep, vals)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(q,)) for q in range(nranks)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errs, errs
    return out


def _sharded_geometry():
    # d < N: the column-orientation Gram, the row-sharded path
    return W.lattice_box(512, 24.0, [dict(cells=(12, 12, 12), step=(1, 1, 1))], M=10,
                         n_vacancies=12, n_impurities=6, q_range=(0.0, 2.0), eps=1e-7, seed=5,
                         name="shard")


@pytest.mark.parametrize("nranks", [2, 3])
def test_row_sharded_rhosvd_matches_single_rank(ctx, nranks):
    g = _sharded_geometry()
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    assert all(d < n for d, n in zip(can.dict_cols, g.N))
    t1, rep1 = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    ranks_out = _run_ranks(g, nranks)
    pr = O.probes(g.N, 400, 3)
    want = t1.entries(pr)
    oref = O.reference(g)
    F, w = O.side_matrices(oref, g)
    orc = O.rhosvd(F, w, eps=g.eps, with_norm=False)
    v_orc = O.projected_cp_entries(w, orc.Z, orc.P, pr)
    for q, (cq, canq, tq, repq) in enumerate(ranks_out):
        assert tuple(repq.chosen_ranks) == tuple(rep1.chosen_ranks) == tuple(orc.ranks)
        for l in range(3):
            s1, sq = rep1.singular_values[l], repq.singular_values[l]
            # the sharded run's eigensolves are cuSOLVER's (owner-solved), the single run's
            # the in-house solver's: the spectra agree to rounding of the smallest values
            assert np.max(np.abs(s1 - sq)) <= 1e-11 * s1[0]
        got = tq.entries(pr)
        scale = np.max(np.abs(want))
        assert np.max(np.abs(got - want)) / scale < 1e-11, q  # same tensor, other summation order
        assert np.max(np.abs(got - v_orc)) / np.max(np.abs(v_orc)) <= 10 * g.eps + 1e-12
        np.testing.assert_allclose(repq.input_norm, rep1.input_norm, rtol=1e-12)
    # every rank holds the full, identical result (Z all-gathered, core all-reduced)
    cores = [o[2].core for o in ranks_out]
    for c in cores[1:]:
        assert np.array_equal(c, cores[0])


def test_row_sharded_full_cfg3_against_fixture():
    """BASELINE cfg3 at full size on two ranks: the randomized second pass and the
    distributed pass-1 eigensolves (rank q solves mode q, the others receive) in the
    sharded path, against the oracle fixture."""
    path = os.path.join(os.path.dirname(__file__), "golden", "fullcfg3.npz")
    fx = np.load(path)
    g = W.baseline(3)
    out = _run_ranks(g, 2)
    for _, _, t, rep in out:
        assert list(rep.chosen_ranks) == list(fx["ranks"])
        pr = fx["probes"]
        v = t.entries(pr)
        assert np.max(np.abs(v - fx["v_rhosvd"])) / np.max(np.abs(fx["v_rhosvd"])) <= 10 * g.eps + 1e-12
    assert np.array_equal(out[0][2].core, out[1][2].core)


@pytest.fixture(autouse=True)
def _finite_collectives(monkeypatch):
    """Everything a rank hands to a collective is finite: a buffer with tiles nobody wrote (the
    upper triangle of a lower-only SYRK, once) would be summed as whatever the pool held."""
    orig_ar, orig_ag = api.ThreadCollective.allreduce, api.ThreadCollective.allgather

    def allreduce(self, rank, channel, buf):
        assert np.all(np.isfinite(buf)), (rank, channel, buf.size)
        return orig_ar(self, rank, channel, buf)

    def allgather(self, rank, channel, send, recv):
        assert np.all(np.isfinite(send)), (rank, channel, send.size)
        return orig_ag(self, rank, channel, send, recv)

    monkeypatch.setattr(api.ThreadCollective, "allreduce", allreduce)
    monkeypatch.setattr(api.ThreadCollective, "allgather", allgather)
    yield


@pytest.mark.parametrize("nranks", [2, 3])
def test_core_slabs_match_the_full_core(ctx, nranks):
    """SURVEY 8e's per-rank core slabs (LATSUM_RHOSVD_CORE_SLABS): each rank forms rows
    [r1 q/P, r1 (q+1)/P) of mode 1 over the whole contraction, no core all-reduce; stacked,
    the slabs are the single-rank core, and entries / boxes (partials + all-reduce) match."""
    g = _sharded_geometry()
    ref = api.reference_for(g, ctx)
    can = api.lattice_sum(ref, g)
    t1, rep1 = api.rhosvd(can, api.TruncationSpec.tol(g.eps))
    full = t1.core
    box = ((100, 200, 250), (140, 260, 262))
    want_box = t1.to_dense(*box)
    outs = _run_ranks(g, nranks, core_slabs=True, box=box)
    slabs = []
    for q, (cq, canq, tq, repq, vals) in enumerate(outs):
        assert tuple(repq.chosen_ranks) == tuple(rep1.chosen_ranks)
        a0, slab = tq.core_slab()
        assert a0 == full.shape[0] * q // nranks
        slabs.append(slab)
        with pytest.raises(Exception):
            tq.core  # the whole core lives on no rank
        scale = np.max(np.abs(want_box))
        assert np.max(np.abs(vals - want_box)) / scale < 1e-11
        pr = O.probes(g.N, 200, 9)
        v1 = t1.entries(pr)
        # every rank gets the summed values (collective: the other ranks evaluate too)
        assert vals.shape == want_box.shape
    # the core depends on the bases' signs: compare with the all-reduced core of a sharded
    # run without slabs (same owner-solved bases)
    ref_core = _run_ranks(g, nranks)[0][2].core
    stacked = np.concatenate(slabs, axis=0)
    assert stacked.shape == ref_core.shape == full.shape
    assert np.max(np.abs(stacked - ref_core)) <= 1e-12 * np.max(np.abs(ref_core))
