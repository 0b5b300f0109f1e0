"""world_size-2 gloo checks of the multi-GPU decomposition (CPU, no GPU needed).

The CUDA path shards RHOSVD over grid rows (latsum_capi.cu reduce_mode): every
contraction over the grid index is a partial product followed by an all-reduce,
eigensolves run redundantly, Z is all-gathered, and the evaluation box is split into
z-slabs.  Here two gloo ranks run the same sequence of partial products and
all-reduces in numpy and must reproduce the single-process oracle: identical ranks,
singular values, and reconstructed values."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1411_1994_b200 import workload as W
from latsum_helpers import mini


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(a: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(a))
    dist.all_reduce(t)
    return t.numpy()


def _polar(U, iters=2):
    for _ in range(iters):
        S = _allreduce(U.T @ U)
        U = 1.5 * U - 0.5 * U @ S
    return U


def _sharded_mode(sd, eps, rank, world):
    """Mirror of reduce_mode's column orientation with the rows [lo, hi) of this rank."""
    N, d = sd.rows, sd.U.shape[1]
    lo, hi = W.row_block(N, rank, world)
    At = (sd.U * np.sqrt(sd.counts)[None, :])[lo:hi]
    G = _allreduce(At.T @ At)
    lam, V = np.linalg.eigh(G)
    lam_d = np.maximum(lam[::-1], 0.0)
    n = d
    k1 = max(int(np.sum(lam_d > 1e-10 * lam_d[0])), 1)
    nc = n - k1
    U1 = _polar(At @ V[:, ::-1][:, :k1] / np.sqrt(lam_d[:k1])[None, :])
    Ap = At.copy()
    for _ in range(2):
        C = _allreduce(U1.T @ Ap)
        Ap = Ap - U1 @ C
    Qc = V[:, :nc]
    B = Ap @ Qc
    mu, Wv = np.linalg.eigh(_allreduce(B.T @ B))
    mu_d = np.maximum(mu[::-1], 0.0)
    allv = sorted([(lam_d[i], 0, i) for i in range(k1)] + [(mu_d[i], 1, i) for i in range(nc)],
                  key=lambda x: -x[0])
    merged = np.array([a[0] for a in allv])
    n_sing = min(N, sd.cols)
    sv = np.zeros(n_sing)
    sv[:min(n_sing, n)] = np.sqrt(merged[:min(n_sing, n)])
    r = O.rank_for_tolerance(sv, eps)
    while r > 1 and sv[r - 1] < 1e-14 * sv[0]:
        r -= 1
    need2 = max([a[2] + 1 for a in allv[:r] if a[1] == 1], default=0)
    cols = [U1]
    if need2:
        cols.append(_polar(B @ Wv[:, ::-1][:, :need2] / np.sqrt(mu_d[:need2])[None, :]))
    cat = np.concatenate(cols, axis=1)
    sel = [a[2] if a[1] == 0 else k1 + a[2] for a in allv[:r]]
    Zb = cat[:, sel]
    P = _allreduce(Zb.T @ sd.U[lo:hi])        # P_l = Z_l^T D_l over rows, summed
    blocks = [torch.zeros(0)] * world
    parts = [torch.zeros((W.row_block(N, q, world)[1] - W.row_block(N, q, world)[0]) * r,
                         dtype=torch.float64) for q in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(Zb.T).ravel()))
    Z = np.concatenate([p.numpy().reshape(r, -1).T for p in parts], axis=0)
    return r, sv, Z, O.ProjectedFactor(P, sd.inv)


def _worker(rank, world, port, kind, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g = mini(kind)
    ref = O.reference(g)
    sides, w = O.side_dictionary(ref, g)
    res = [_sharded_mode(sides[l], g.eps, rank, world) for l in range(3)]
    if rank == 0:
        pr = O.probes(g.N, 200, 5)
        v = O.projected_cp_entries(w, [x[2] for x in res], [x[3] for x in res], pr)
        np.savez(os.path.join(out_dir, f"{kind}.npz"), ranks=np.array([x[0] for x in res]),
                 s0=res[0][1], s1=res[1][1], s2=res[2][1], v=v, probes=pr)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["vacancies", "mixed"])
def test_row_sharded_rhosvd_matches_single_process(tmp_path, kind):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), kind, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(tmp_path / f"{kind}.npz")
    g = mini(kind)
    ref = O.reference(g)
    sides, w = O.side_dictionary(ref, g)
    orc = O.rhosvd(sides, w, eps=g.eps, with_norm=False)
    assert tuple(got["ranks"]) == tuple(orc.ranks)
    for l in range(3):
        s = got[f"s{l}"]
        assert np.max(np.abs(s - orc.sigma[l])) / orc.sigma[l][0] < 1e-10
    want = O.projected_cp_entries(w, orc.Z, orc.P, got["probes"])
    assert np.max(np.abs(got["v"] - want)) / np.max(np.abs(want)) <= 10 * g.eps + 1e-12


def test_z_slabs_partition_the_box():
    lo, hi = (3, 5, 7), (40, 41, 1031)
    for world in (1, 2, 3, 8):
        zs = []
        for r in range(world):
            a, b = W.z_slab(lo, hi, r, world)
            assert a[:2] == lo[:2] and b[:2] == hi[:2]
            zs.extend(range(a[2], b[2]))
        assert zs == list(range(lo[2], hi[2]))


def test_row_blocks_partition_rows():
    for n in (1, 7, 2048, 32768):
        for world in (1, 2, 4, 8):
            rows = []
            for r in range(world):
                a, b = W.row_block(n, r, world)
                rows.extend(range(a, b))
            assert rows == list(range(n))


def _collective_worker(rank, world, port, out_dir):
    """The library's host-collective callbacks over gloo (api.TorchCollective): concurrent
    channels from several threads, as the library's worker streams call them."""
    import threading
    from paper_1411_1994_b200 import api
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    coll = api.TorchCollective()
    res = {}

    def channel(ch):
        rng = np.random.default_rng(100 * ch + rank)
        for it in range(5):
            a = rng.standard_normal(37 + it)
            b = a.copy()
            coll.allreduce(rank, ch, b)
            g = np.zeros(world * a.size)
            coll.allgather(rank, ch, a, g)
            res[(ch, it)] = (a, b, g)

    th = [threading.Thread(target=channel, args=(ch,)) for ch in range(5)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    np.savez(os.path.join(out_dir, f"coll{rank}.npz"),
             **{f"{k[0]}_{k[1]}_{i}": v[i] for k, v in res.items() for i in range(3)})
    dist.barrier()
    dist.destroy_process_group()


def test_host_collective_over_gloo(tmp_path):
    world = 2
    mp.start_processes(_collective_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    f = [np.load(tmp_path / f"coll{r}.npz") for r in range(world)]
    for ch in range(5):
        for it in range(5):
            a = [f[r][f"{ch}_{it}_0"] for r in range(world)]
            for r in range(world):
                np.testing.assert_allclose(f[r][f"{ch}_{it}_1"], a[0] + a[1], rtol=1e-15)
                assert np.array_equal(f[r][f"{ch}_{it}_2"], np.concatenate(a))
            assert np.array_equal(f[0][f"{ch}_{it}_1"], f[1][f"{ch}_{it}_1"])  # bit-identical
