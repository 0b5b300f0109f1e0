"""GPU eigensolver building blocks (csrc/eig_sym.cuh) against numpy LAPACK.

The custom symmetric eigensolver replaces cuSOLVER syevd for the RHOSVD Grams; each stage
is checked on Gram-like matrices whose spectra decay over 16 decades (as the side-matrix
Grams do) and on random symmetric matrices with both signs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gram_like(n, seed, decades=16.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))
    return (Q * lam) @ Q.T


def _sym(n, seed):
    rng = np.random.default_rng(seed)
    B = rng.standard_normal((n, n))
    return (B + B.T) / 2


def _sytrd(ctx, A):
    import torch
    from paper_1411_1994_b200 import _lib
    n = A.shape[0]
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
    d = torch.zeros(n, dtype=torch.float64, device="cuda")
    e = torch.zeros(max(n - 1, 1), dtype=torch.float64, device="cuda")
    tau = torch.zeros(max(n - 1, 1), dtype=torch.float64, device="cuda")
    ctx.check(_lib.lib().latsum_sytrd_device(ctx.handle, n, dA.data_ptr(), n, d.data_ptr(),
                                             e.data_ptr(), tau.data_ptr()))
    ctx.synchronize()
    return (dA.cpu().numpy().reshape((n, n), order="F"), d.cpu().numpy(),
            e.cpu().numpy()[: n - 1], tau.cpu().numpy()[: n - 1])


def _q_from_reflectors(Af, tau):
    n = Af.shape[0]
    Q = np.eye(n)
    for k in range(n - 2, -1, -1):
        v = np.zeros(n)
        v[k + 1] = 1.0
        v[k + 2:] = Af[k + 2:, k]
        Q -= tau[k] * np.outer(v, v @ Q)
    return Q


@pytest.mark.parametrize("n", [1, 2, 3, 5, 33, 100, 357, 693, 1100])
@pytest.mark.parametrize("kind", ["gram", "sym"])
def test_sytrd_cluster_matches_lapack(ctx, n, kind):
    A = _gram_like(n, n) if kind == "gram" else _sym(n, n + 1)
    Af, d, e, tau = _sytrd(ctx, A)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    scale = np.linalg.norm(A, 2)
    lam_t = np.linalg.eigvalsh(T)
    lam_a = np.linalg.eigvalsh(A)
    assert np.max(np.abs(lam_t - lam_a)) <= 1e-13 * max(scale, 1e-300) * max(1, np.sqrt(n) / 4)
    Q = _q_from_reflectors(Af, tau)
    assert np.max(np.abs(Q.T @ Q - np.eye(n))) < 1e-13 * max(1, np.sqrt(n) / 4)
    assert np.max(np.abs(Q @ T @ Q.T - A)) <= 1e-13 * max(scale, 1e-300) * max(1, np.sqrt(n) / 4)


@pytest.mark.parametrize("n", [2, 3, 40, 357, 693, 1200])
@pytest.mark.parametrize("kind", ["gram", "sym"])
def test_eigensolver_matches_lapack(ctx, n, kind):
    """Eigenvalues (all) and the leading eigenvectors of the in-house solver vs numpy eigh:
    |lam - lam_ref| <= 1e-13 ||A||; the leading vectors (well separated in the Gram-like
    spectra: the top third) match up to sign to eps ||A|| / gap and are orthonormal."""
    import torch
    from paper_1411_1994_b200 import _lib
    A = _gram_like(n, n + 7) if kind == "gram" else _sym(n, n + 8)
    k = max(1, n // 3)
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
    w = torch.zeros(n, dtype=torch.float64, device="cuda")
    V = torch.zeros(n * k, dtype=torch.float64, device="cuda")
    ctx.check(_lib.lib().latsum_eig_sym_device(ctx.handle, n, dA.data_ptr(), k, w.data_ptr(),
                                               V.data_ptr(), 2))
    lam = w.cpu().numpy()
    Vh = V.cpu().numpy().reshape((n, k), order="F")
    lr, vr = np.linalg.eigh(A)
    scale = np.abs(lr).max()
    assert np.max(np.abs(lam - lr)) <= 1e-13 * scale * max(1.0, np.sqrt(n) / 8)
    order = np.argsort(lr)[::-1][:k]
    for j in range(k):
        lj = lr[order[j]]
        gap = np.min(np.abs(np.delete(lr, order[j]) - lj)) if n > 1 else scale
        v = vr[:, order[j]]
        err = min(np.linalg.norm(Vh[:, j] - v), np.linalg.norm(Vh[:, j] + v))
        assert err <= 1e-12 + 64 * 2.2e-16 * scale * np.sqrt(n) / max(gap, 1e-300), (j, err, gap)
    if kind == "sym":  # well-separated random spectrum: numerically orthonormal
        assert np.max(np.abs(Vh.T @ Vh - np.eye(k))) < 1e-10


@pytest.mark.parametrize("n", [2, 3, 5, 17, 18, 19, 33, 40, 100, 357, 693, 808])
@pytest.mark.parametrize("kind", ["gram", "sym"])
def test_band_eigensolver_matches_lapack(ctx, n, kind):
    """Two-stage solver (full -> band in one cluster, bulge chasing in shared memory,
    inverse iteration, fused back-transform) vs numpy eigh, same bounds as above."""
    import torch
    from paper_1411_1994_b200 import _lib
    A = _gram_like(n, n + 17) if kind == "gram" else _sym(n, n + 18)
    k = max(1, n // 3)
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
    w = torch.zeros(n, dtype=torch.float64, device="cuda")
    V = torch.zeros(n * k, dtype=torch.float64, device="cuda")
    ctx.check(_lib.lib().latsum_eig_sym_device(ctx.handle, n, dA.data_ptr(), k, w.data_ptr(),
                                               V.data_ptr(), 3))
    lam = w.cpu().numpy()
    Vh = V.cpu().numpy().reshape((n, k), order="F")
    lr, vr = np.linalg.eigh(A)
    scale = np.abs(lr).max()
    assert np.max(np.abs(lam - lr)) <= 1e-13 * scale * max(1.0, np.sqrt(n) / 8)
    order = np.argsort(lr)[::-1][:k]
    for j in range(k):
        lj = lr[order[j]]
        gap = np.min(np.abs(np.delete(lr, order[j]) - lj)) if n > 1 else scale
        v = vr[:, order[j]]
        err = min(np.linalg.norm(Vh[:, j] - v), np.linalg.norm(Vh[:, j] + v))
        assert err <= 1e-12 + 64 * 2.2e-16 * scale * np.sqrt(n) / max(gap, 1e-300), (j, err, gap)
    if kind == "sym":
        assert np.max(np.abs(Vh.T @ Vh - np.eye(k))) < 1e-10
