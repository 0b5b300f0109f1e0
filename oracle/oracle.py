"""latsum CPU ORACLE driver — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module, and only as the checker.  The
product package never imports it.

It restates the reference pipeline on the CPU on top of latsum_oracle.cpp
(C++ restatement of the per-entry loops) and numpy/LAPACK (the SVD that
Eigen's BDCSVD performs in the reference):

* `reference`         reference.hpp:95-153 build_reference_canonical
* `side_matrices`     lattice_sum.hpp:198-223 assembled_sum_canonical, :148-157
                      windowed_canonical, :339-384 defected_sum (canonical
                      branch, add_concat order), :411-465 sublattice_union_sum
* `rhosvd`            rank_reduction.hpp:176-218 (+ :73-84 rank_for_tolerance,
                      :88-100 project_core, :61-66 tail)
* `oracle_entries`    lattice_sum.hpp:656-671 oracle_entry (brute force)

PARITY PINNED against the reference itself: oracle/_ref (the reference's headers compiled
against the stand-ins of oracle/shim, driven by oracle/ref.py) and its golden vectors
tests/golden/refpin_*.npz; see tests/test_reference_pin.py.

The SVD runs on the column-merged side matrix (identical columns merged with
sqrt(multiplicity) weights), which has the same A A^T, left singular vectors
and nonzero singular values as the reference's N x M_c matrix.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblatsum_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "latsum_oracle.cpp"))):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        d, i, i64, p = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        L.orc_build_quadrature.argtypes = [i, d, i, d, d, d, p, p]
        L.orc_build_quadrature.restype = i
        L.orc_default_step_constant.argtypes = [i, d, i, d, d, i]
        L.orc_default_step_constant.restype = d
        L.orc_shell_error.argtypes = [i, d, p, p, i, d, d, i]
        L.orc_shell_error.restype = d
        L.orc_mode_integrals.argtypes = [p, i, i64, d, d, i, p]
        L.orc_normalize_columns.argtypes = [i64, i64, p, p]
        L.orc_assembled_vector.argtypes = [p, i64, p, i64, p]
        L.orc_assembled_vector.restype = i64
        L.orc_assembled_vector_sliding.argtypes = [p, i64, i64, i64, i, i, p]
        L.orc_canonical_entries.argtypes = [p, i64, p, p, p, p, p, i64, p]
        L.orc_tucker_entries.argtypes = [p, p, p, p, p, p, p, i64, p]
        L.orc_oracle_entries.argtypes = [p, i64, p, p, p, p, p, p, i64, p, i64, p, i]
        L.orc_project_core.argtypes = [p, i64, p, p, p, p, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _f64F(a) -> np.ndarray:
    return np.asfortranarray(a, dtype=np.float64)


# ----------------------------------------------------------------------------- stage 1

def quadrature(family: int, lam: float, M: int, C0: float, a: float, A: float):
    R = 2 * M + 1
    nodes, weights = np.zeros(R), np.zeros(R)
    if lib().orc_build_quadrature(family, lam, M, C0, a, A, _ptr(nodes), _ptr(weights)):
        raise ValueError("build_quadrature: M >= 2, 0 < a < A, C0 > 0 required")
    return nodes, weights


def default_step_constant(family: int, lam: float, M: int, a: float, A: float,
                          npts: int = 320) -> float:
    return lib().orc_default_step_constant(family, lam, M, a, A, npts)


def reference_shell(N, box):
    """reference.hpp:84-93 on the doubled grid (mesh h, box 2b)."""
    hmin = min(float(b) / float(n) for b, n in zip(box, N))
    bmax = max(2.0 * float(b) for b in box)
    return hmin, float(np.sqrt(3.0)) * bmax / 2.0


def mode_integrals(nodes, n2: int, lower: float, h: float, variant: str = "hybrid"):
    nodes = _f64(nodes)
    out = np.zeros((n2, nodes.size), order="F")
    lib().orc_mode_integrals(_ptr(nodes), nodes.size, n2, lower, h,
                             1 if variant == "hybrid" else 0, _ptr(out))
    return out


def normalize_columns(m: np.ndarray):
    m = _f64F(m).copy(order="F")
    norms = np.zeros(m.shape[1])
    lib().orc_normalize_columns(m.shape[0], m.shape[1], _ptr(m), _ptr(norms))
    return m, norms


@dataclass
class RefOracle:
    N: tuple
    box: tuple
    M: int
    C0: float
    shell: tuple
    nodes: np.ndarray
    quad_weights: np.ndarray
    factors: List[np.ndarray]  # 3 x (2N_l x R), unit columns
    weights: np.ndarray  # R


def reference(geom, variant: str = "hybrid") -> RefOracle:
    """reference.hpp:95-153 for a single primitive (coefficient 1)."""
    N, box = tuple(geom.N), tuple(geom.box)
    a, A = reference_shell(N, box)
    C0 = geom.C0 if geom.C0 > 0 else default_step_constant(geom.family, geom.lam, geom.M, a, A)
    nodes, qw = quadrature(geom.family, geom.lam, geom.M, C0, a, A)
    weights = 1.0 * qw  # coefficient * rule weight
    raw = []
    for l in range(3):
        same = None
        for m in range(l):
            if N[l] == N[m] and box[l] == box[m]:
                same = m
                break
        if same is not None:
            raw.append(raw[same].copy(order="F"))
        else:
            h = float(box[l]) / float(N[l])  # doubled grid: 2b / 2N
            raw.append(mode_integrals(nodes, 2 * N[l], -float(box[l]), h, variant))
    factors = []
    w = weights.copy()
    for l in range(3):  # canonical.hpp:32-48 from_raw
        f, nrm = normalize_columns(raw[l])
        for q in range(w.size):
            if nrm[q] == 0.0:
                w[q] = 0.0
            else:
                w[q] *= nrm[q]
        factors.append(f)
    return RefOracle(N, box, geom.M, C0, (a, A), nodes, qw, factors, w)


# ----------------------------------------------------------------------------- stage 2

def assembled_vector(ref_col: np.ndarray, N: int, shifts: np.ndarray) -> np.ndarray:
    out = np.zeros(N)
    sh = np.ascontiguousarray(shifts, dtype=np.int64)
    bad = lib().orc_assembled_vector(_ptr(_f64(ref_col)), N, _ptr(sh), sh.size, _ptr(out))
    if bad:
        raise OverflowError(f"window overflow: shift {int(sh[bad - 1])}")
    return out


def side_matrix_mode(ref: RefOracle, geom, l: int):
    """One mode of `side_matrices`: the N_l x M_c unit-column side matrix in reference
    column order and the per-column norms that from_raw folds into the weights (the
    reference builds every block's columns this way: assembled_vector / windowed
    columns, lattice_sum.hpp:101-157, then canonical.hpp:32-48)."""
    N, R = geom.N[l], geom.R
    blocks = geom.blocks()
    F = np.zeros((N, R * len(blocks)), order="F")
    norms = np.zeros(R * len(blocks))
    for b, blk in enumerate(blocks):
        raw = np.zeros((N, R), order="F")
        for q in range(R):
            raw[:, q] = assembled_vector(ref.factors[l][:, q], N, blk.shifts[l])
        f, nrm = normalize_columns(raw)
        F[:, b * R:(b + 1) * R] = f
        norms[b * R:(b + 1) * R] = nrm
    return F, norms


def side_matrices(ref: RefOracle, geom, max_bytes: float = 24e9):
    """Full N x M_c side matrices in reference column order + M_c weights.

    Blocks: every sublattice (assembled, R columns), then every defect
    (windowed, R columns), each block normalised by from_raw.
    """
    N, R = geom.N, geom.R
    Mc = geom.canonical_rank
    if 8.0 * Mc * sum(N) > max_bytes:
        raise MemoryError("side matrices exceed the oracle's memory budget")
    F = [np.zeros((N[l], Mc), order="F") for l in range(3)]
    w = np.zeros(Mc)
    col = 0
    blocks = [(b.shifts, b.charge) for b in geom.blocks()]
    for shifts, charge in blocks:
        wb = charge * ref.weights
        for l in range(3):
            raw = np.zeros((N[l], R), order="F")
            for q in range(R):
                raw[:, q] = assembled_vector(ref.factors[l][:, q], N[l], shifts[l])
            f, nrm = normalize_columns(raw)
            for q in range(R):
                wb[q] = 0.0 if nrm[q] == 0.0 else wb[q] * nrm[q]
            F[l][:, col:col + R] = f
        w[col:col + R] = wb
        col += R
    return F, w


# ----------------------------------------------------------------------------- stage 3

def merge_columns(F: np.ndarray):
    """Unique columns (exact equality) with multiplicities and inverse map."""
    seen = {}
    inv = np.zeros(F.shape[1], np.int64)
    uniq = []
    for q in range(F.shape[1]):
        key = F[:, q].tobytes()
        j = seen.get(key)
        if j is None:
            j = len(uniq)
            seen[key] = j
            uniq.append(q)
        inv[q] = j
    U = F[:, uniq]
    counts = np.bincount(inv, minlength=len(uniq)).astype(np.float64)
    return np.asfortranarray(U), counts, inv


def rank_for_tolerance(sv: np.ndarray, eps: float) -> int:
    """rank_reduction.hpp:73-84."""
    target = eps * float(np.linalg.norm(sv)) / 3.0
    tail2 = 0.0
    r = sv.size
    for k in range(sv.size - 1, -1, -1):
        tail2 += sv[k] * sv[k]
        if np.sqrt(tail2) > target:
            break
        r = k
    return max(r, 1)


def input_norm(F, w, chunk: int = 4096) -> float:
    """canonical.hpp:148-162 norm_f via the Hadamard of the three Grams, on
    merged identical terms and unique columns (same value)."""
    uniq, inv = [], []
    for l in range(3):
        U, _, iv = merge_columns(F[l])
        uniq.append(U)
        inv.append(iv)
    key = np.stack(inv, axis=1)
    terms, tinv = np.unique(key, axis=0, return_inverse=True)
    wt = np.bincount(tinv.ravel(), weights=w, minlength=terms.shape[0])
    G = [uniq[l].T @ uniq[l] for l in range(3)]
    s = 0.0
    T = terms.shape[0]
    for a in range(0, T, chunk):
        ia = terms[a:a + chunk]
        blk = (G[0][np.ix_(ia[:, 0], terms[:, 0])] * G[1][np.ix_(ia[:, 1], terms[:, 1])]
               * G[2][np.ix_(ia[:, 2], terms[:, 2])])
        s += float(wt[a:a + chunk] @ (blk @ wt))
    return float(np.sqrt(s)) if s > 0 else 0.0


@dataclass
class RhosvdOracle:
    sigma: List[np.ndarray]
    ranks: tuple
    Z: List[np.ndarray]
    P: List[np.ndarray]  # Z^T A_l over the full M_c columns
    tie: tuple
    weight_norm: float
    input_norm: Optional[float]
    bound_abs: float
    bound_rel: Optional[float]
    stability_constant: Optional[float]
    margin: tuple  # (tail(r) - target) / target style cutoff margins


@dataclass
class DictSide:
    """One mode's side matrix in merged form: F = U[:, inv] (unique columns U,
    multiplicities counts)."""
    U: np.ndarray
    counts: np.ndarray
    inv: np.ndarray
    rows: int
    cols: int  # M_c


def side_dictionary(ref: RefOracle, geom):
    """Memory-light form of `side_matrices`: each distinct (placement, reference column)
    is assembled and normalised once (lattice_sum.hpp:101-157 + canonical.hpp:32-48) —
    the same columns, bit for bit, that the full N x M_c matrices hold — plus the M_c
    weights in reference order (sublattice blocks, then defects)."""
    N, R = geom.N, geom.R
    blocks = [(tuple(np.asarray(x, np.int64) for x in b.shifts), b.charge)
              for b in geom.blocks()]
    Mc = R * len(blocks)
    w = np.zeros(Mc)
    sides = []
    norms_l = []
    for l in range(3):
        _, _, rinv = merge_columns(ref.factors[l])  # distinct reference columns
        rep_col = {}
        for k in range(R):
            rep_col.setdefault(int(rinv[k]), k)
        cols, norms, key_to_col = [], [], {}
        inv = np.zeros(Mc, np.int64)
        for b, (shifts, _) in enumerate(blocks):
            pkey = shifts[l].tobytes()
            for k in range(R):
                key = (pkey, int(rinv[k]))
                j = key_to_col.get(key)
                if j is None:
                    v = assembled_vector(ref.factors[l][:, rep_col[int(rinv[k])]], N[l], shifts[l])
                    f, nv = normalize_columns(v.reshape(-1, 1))
                    j = len(cols)
                    key_to_col[key] = j
                    cols.append(f[:, 0].copy())
                    norms.append(float(nv[0]))
                inv[b * R + k] = j
        U = np.asfortranarray(np.stack(cols, axis=1))
        counts = np.bincount(inv, minlength=U.shape[1]).astype(np.float64)
        sides.append(DictSide(U, counts, inv, N[l], Mc))
        norms_l.append(np.asarray(norms))
    for b, (_, charge) in enumerate(blocks):
        wb = charge * ref.weights
        for l in range(3):
            nv = norms_l[l][sides[l].inv[b * R:(b + 1) * R]]
            wb = np.where(nv == 0.0, 0.0, wb * nv)
        w[b * R:(b + 1) * R] = wb
    return sides, w


def as_dict_sides(F):
    out = []
    for f in F:
        U, counts, inv = merge_columns(f)
        out.append(DictSide(U, counts, inv, f.shape[0], f.shape[1]))
    return out


def rhosvd(F, w, eps: Optional[float] = None, ranks=None, with_norm: bool = True) -> RhosvdOracle:
    """rank_reduction.hpp:176-218 on the merged-column SVD.  F is either the three full
    N x M_c side matrices or their `DictSide` forms (same result)."""
    sides = F if isinstance(F[0], DictSide) else as_dict_sides(F)
    sig, Zs, rk, tie, Ps, margins = [], [], [], [], [], []
    for l in range(3):
        sd = sides[l]
        Ad = sd.U * np.sqrt(sd.counts)[None, :]
        u, s, _ = np.linalg.svd(Ad, full_matrices=False)
        n_full = min(sd.rows, sd.cols)
        sv = np.zeros(n_full)
        sv[:s.size] = s
        if ranks is not None:
            r = min(int(ranks[l]), sv.size)
        else:
            r = rank_for_tolerance(sv, eps)
        while r > 1 and sv[r - 1] < 1e-14 * sv[0]:
            r -= 1
        tie.append(bool(r < sv.size and sv[r - 1] - sv[r] <= 1e-12 * sv[0]))
        if eps is not None:
            target = eps * np.linalg.norm(sv) / 3.0
            t_r = np.sqrt(np.sum(sv[r:] ** 2))
            t_rm1 = np.sqrt(np.sum(sv[r - 1:] ** 2))
            margins.append(float(min(target - t_r, t_rm1 - target) / target))
        sig.append(sv)
        rk.append(r)
        Z = np.asfortranarray(u[:, :r])
        del u
        Zs.append(Z)
        Ps.append(ProjectedFactor(np.asfortranarray(Z.T @ sd.U), sd.inv))
    wn = float(np.linalg.norm(w))
    tails = sum(float(np.sqrt(np.sum(sig[l][rk[l]:] ** 2))) for l in range(3))
    nrm = input_norm_dict(sides, w) if with_norm else None
    stab = (wn * wn / (nrm * nrm)) if nrm else None
    brel = (np.sqrt(stab) * nrm * tails) if nrm else None
    return RhosvdOracle(sig, tuple(rk), Zs, Ps, tuple(tie), wn, nrm, wn * tails, brel, stab,
                        tuple(margins))


class ProjectedFactor:
    """P_l = Z_l^T A_l (r x M_c) stored as Z_l^T U_l and the column map."""

    def __init__(self, Pu, inv):
        self.Pu, self.inv = Pu, inv

    @property
    def shape(self):
        return (self.Pu.shape[0], self.inv.size)

    def full(self):
        return np.asfortranarray(self.Pu[:, self.inv])

    def __getitem__(self, idx):
        return self.full()[idx]

    def __array__(self, dtype=None, copy=None):
        return self.full()


def input_norm_dict(sides, w, chunk: int = 4096) -> float:
    """canonical.hpp:148-162 via unique-column Grams and merged identical terms."""
    key = np.stack([sd.inv for sd in sides], axis=1)
    terms, tinv = np.unique(key, axis=0, return_inverse=True)
    wt = np.bincount(tinv.ravel(), weights=w, minlength=terms.shape[0])
    G = [sd.U.T @ sd.U for sd in sides]
    s = 0.0
    T = terms.shape[0]
    for a in range(0, T, chunk):
        ia = terms[a:a + chunk]
        blk = (G[0][np.ix_(ia[:, 0], terms[:, 0])] * G[1][np.ix_(ia[:, 1], terms[:, 1])]
               * G[2][np.ix_(ia[:, 2], terms[:, 2])])
        s += float(wt[a:a + chunk] @ (blk @ wt))
    return float(np.sqrt(s)) if s > 0 else 0.0


def project_core(w, P) -> np.ndarray:
    """rank_reduction.hpp:88-100 (reference loop order; small sizes only)."""
    p = [_f64F(x.full() if isinstance(x, ProjectedFactor) else x) for x in P]
    r = np.array([p[0].shape[0], p[1].shape[0], p[2].shape[0]], np.int64)
    core = np.zeros(int(np.prod(r)))
    lib().orc_project_core(_ptr(_f64(w)), p[0].shape[1], _ptr(p[0]), _ptr(p[1]), _ptr(p[2]),
                           _ptr(r), _ptr(core))
    return core.reshape(tuple(r), order="F")


# ----------------------------------------------------------------------------- entries

def canonical_entries(F, w, probes: np.ndarray) -> np.ndarray:
    """canonical.hpp:63-70 at probes (full side matrices or DictSide forms)."""
    pr = np.ascontiguousarray(probes, dtype=np.int64)
    rows = []
    for l in range(3):
        if isinstance(F[l], DictSide):
            rows.append(F[l].U[pr[:, l]][:, F[l].inv])
        else:
            rows.append(F[l][pr[:, l]])
    return np.einsum("q,pq,pq,pq->p", w, rows[0], rows[1], rows[2])


def projected_cp_entries(w, Z, P, probes: np.ndarray) -> np.ndarray:
    """Tucker value of the RHOSVD result at probes via the projected-CP identity
    V = sum_q w_q prod_l (Z_l Z_l^T a_lq)(i_l); equals TuckerTensor::entry."""
    pr = np.ascontiguousarray(probes, dtype=np.int64)
    Q = []
    for l in range(3):
        if isinstance(P[l], ProjectedFactor):
            Q.append((Z[l][pr[:, l]] @ P[l].Pu)[:, P[l].inv])
        else:
            Q.append(Z[l][pr[:, l]] @ P[l])
    return (Q[0] * Q[1] * Q[2]) @ w


def tucker_entries(core, U, probes: np.ndarray) -> np.ndarray:
    """tucker.hpp:38-54 per probe (C++ loop)."""
    core = _f64F(core)
    r = np.array(core.shape, np.int64)
    dims = np.array([U[0].shape[0], U[1].shape[0], U[2].shape[0]], np.int64)
    u = [_f64F(x) for x in U]
    pr = np.ascontiguousarray(probes, dtype=np.int64)
    out = np.zeros(pr.shape[0])
    lib().orc_tucker_entries(_ptr(np.ascontiguousarray(core.ravel(order="F"))), _ptr(r),
                             _ptr(u[0]), _ptr(u[1]), _ptr(u[2]), _ptr(dims), _ptr(pr),
                             pr.shape[0], _ptr(out))
    return out


def oracle_entries(ref: RefOracle, geom, probes: np.ndarray, threads: int = 0) -> np.ndarray:
    """lattice_sum.hpp:656-671 oracle_entry over all sources (brute force)."""
    shifts, sw = geom.sources()
    pr = np.ascontiguousarray(probes, dtype=np.int64)
    out = np.zeros(pr.shape[0])
    N = np.array(geom.N, np.int64)
    threads = threads or (os.cpu_count() or 1)
    f = [_f64F(x) for x in ref.factors]
    lib().orc_oracle_entries(_ptr(_f64(ref.weights)), ref.weights.size, _ptr(f[0]), _ptr(f[1]),
                             _ptr(f[2]), _ptr(N), _ptr(shifts), _ptr(sw), shifts.shape[0],
                             _ptr(pr), pr.shape[0], _ptr(out), threads)
    return out


def probes(dims, count: int, seed: int) -> np.ndarray:
    """Seeded uniform probe points (commands.cpp:254-266 uses 500 probes)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.stack([rng.integers(0, dims[l], size=count) for l in range(3)], axis=1).astype(
        np.int64)


# ----------------------------------------------------------------------------- canonical_to_tucker

def projected_norm(F, w, Y) -> float:
    """rank_reduction.hpp:104-113."""
    P = [Y[l].T @ F[l] for l in range(3)]
    g = (P[0].T @ P[0]) * (P[1].T @ P[1]) * (P[2].T @ P[2])
    v = float(w @ (g @ w))
    return float(np.sqrt(v)) if v > 0 else 0.0


def als_refine(F, w, Y, ranks, max_sweeps: int = 30, stag_tol: float = 1e-8):
    """rank_reduction.hpp:232-274 (small sizes: full kr unfolding, LAPACK SVD)."""
    Y = [y.copy() for y in Y]
    fit = projected_norm(F, w, Y)
    sweeps = 0
    for _ in range(max_sweeps):
        for l in range(3):
            m1, m2 = (l + 1) % 3, (l + 2) % 3
            p1, p2 = Y[m1].T @ F[m1], Y[m2].T @ F[m2]
            kr = (p1[:, None, :] * p2[None, :, :]).reshape(p1.shape[0] * p2.shape[0], -1) * w[None, :]
            unf = F[l] @ kr.T
            u, _, _ = np.linalg.svd(unf, full_matrices=False)
            Y[l] = np.asfortranarray(u[:, :min(ranks[l], u.shape[1])])
        nxt = projected_norm(F, w, Y)
        sweeps += 1
        if nxt - fit <= stag_tol * max(nxt, 1.0):
            break
        fit = nxt
    return Y, sweeps


def shrink_core(core, factors, budget2, near=None):
    """rank_reduction.hpp:129-168.  `near` (optional list of 3 bools) is set for a mode in
    which some drop decision compared a slice mass within 5% of the initial budget to the
    remaining budget: budget2 = eps^2 n^2 - (n^2 - ||core||^2) carries a cancellation of
    ~1e-16 n^2 / budget2 (percent level at eps = 1e-7), so such a decision is a tie."""
    core = core.copy()
    factors = [f.copy() for f in factors]
    for l in range(3):
        u = np.moveaxis(core, l, 0).reshape(core.shape[l], -1)
        _, q = np.linalg.eigh(u @ u.T)
        q = q[:, ::-1]
        core = np.moveaxis(np.tensordot(q.T, np.moveaxis(core, l, 0), axes=(1, 0)), 0, l)
        factors[l] = factors[l] @ q
    r = list(core.shape)
    budget0 = budget2
    changed = True
    while changed and budget2 > 0:
        changed = False
        for l in range(3):
            if r[l] <= 1:
                continue
            box = core[:r[0], :r[1], :r[2]]
            sl = np.take(box, r[l] - 1, axis=l)
            mass = float(np.sum(sl * sl))
            if near is not None and abs(mass - budget2) <= 0.05 * budget0:
                near[l] = True
            if mass <= budget2:
                budget2 -= mass
                r[l] -= 1
                changed = True
    return core[:r[0], :r[1], :r[2]].copy(), [factors[l][:, :r[l]] for l in range(3)]


def canonical_to_tucker(F, w, eps=None, ranks=None, max_sweeps: int = 30, stag_tol: float = 1e-8,
                        near=None):
    """rank_reduction.hpp:280-306 on full side matrices (small sizes); `near` as in
    shrink_core (tie flags of the slice-drop decisions)."""
    orc = rhosvd(F, w, eps=eps, ranks=ranks, with_norm=True)
    Y, sweeps = als_refine(F, w, orc.Z, orc.ranks, max_sweeps, stag_tol) if max_sweeps > 0 else (orc.Z, 0)
    P = [Y[l].T @ F[l] for l in range(3)]
    core = project_core(w, P)
    if eps is not None and ranks is None:
        n2 = orc.input_norm ** 2
        err2 = max(n2 - float(np.sum(core * core)), 0.0)
        budget2 = eps * eps * n2 - err2
        if budget2 > 0:
            core, Y = shrink_core(core, Y, budget2, near)
    return core, Y, orc, sweeps


# ----------------------------------------------------------------------------- tensor files

def fnv1a64(data: bytes, seed: int = 0xcbf29ce484222325) -> int:
    """tensor_io.cpp:9-17."""
    h = seed
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def tensor_file_bytes(kind: str, dims, payload_u32, arrays) -> bytes:
    """tensor_io.cpp:45-76 write_tensor byte layout ("LTSTNSR" v1, FNV-1a trailer)."""
    import struct
    buf = bytearray(b"LTSTNSR")
    buf += bytes([1, ord(kind), 0, 0, 0])
    buf += struct.pack("<3I", *[int(x) for x in dims])
    buf += struct.pack(f"<{len(payload_u32)}I", *[int(x) for x in payload_u32])
    for a in arrays:
        buf += np.asarray(a, dtype="<f8").ravel(order="F").tobytes()
    buf += struct.pack("<Q", fnv1a64(bytes(buf)))
    return bytes(buf)


# ----------------------------------------------------------------------------- reports

def _g17(x: float) -> str:
    """std::ostream with precision(17), default float format (report.cpp:9-12)."""
    return "%.17g" % float(x)


def spectral_report_text(chosen_ranks, bound_abs, bound_rel, weight_norm, input_norm,
                         stability_constant, stability_ok, tie_at_cutoff, sigma) -> str:
    """report.cpp:28-46 write_spectral_report."""
    out = ["# spectral report\n",
           "chosen_ranks %d %d %d\n" % tuple(int(r) for r in chosen_ranks),
           "bound_abs " + _g17(bound_abs) + "\n", "bound_rel " + _g17(bound_rel) + "\n",
           "weight_norm " + _g17(weight_norm) + "\n", "input_norm " + _g17(input_norm) + "\n",
           "stability_constant " + _g17(stability_constant) + "\n",
           "stability_ok %d\n" % (1 if stability_ok else 0)]
    for l in range(3):
        line = "sigma_mode%d" % (l + 1)
        if tie_at_cutoff[l]:
            line += " (tie at cutoff)"
        line += "".join(" " + _g17(v) for v in sigma[l])
        out.append(line + "\n")
    return "".join(out)


def provenance_text(seed, grid, cells, fmt, rank_or_ranks, summands, bounds=None,
                    extra_lines=()) -> str:
    """report.cpp:48-73 write_provenance (summands: (label, canonical rank, sites))."""
    out = ["# lattice sum provenance\n", "seed %d\n" % seed,
           "grid %d %d %d\n" % tuple(grid), "cells %d %d %d\n" % tuple(cells)]
    if fmt == "canonical":
        out += ["format canonical\n", "rank %d\n" % rank_or_ranks]
    else:
        out += ["format tucker\n", "ranks %d %d %d\n" % tuple(rank_or_ranks)]
    out.append("summands %d\n" % len(summands))
    out += ['summand "%s" rank %d sites %d\n' % (lab, r, s) for lab, r, s in summands]
    if bounds is not None:
        out += ["truncation_bound_abs " + _g17(bounds[0]) + "\n",
                "truncation_bound_rel " + _g17(bounds[1]) + "\n"]
    out += [x + "\n" for x in extra_lines]
    return "".join(out)
