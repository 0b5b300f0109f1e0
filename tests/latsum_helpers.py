"""Shared test helpers (mini geometries mirroring the BASELINE shapes)."""
import numpy as np

from paper_1411_1994_b200 import workload as W


def mini(kind: str, seed: int = 7):
    """Scaled-down versions of the BASELINE configs that the CPU oracle finishes in seconds."""
    if kind == "cubic":        # cfg1 shape: stride-exact cubic lattice, no defects
        return W.lattice_box(64, 8.0, [dict(cells=(4, 4, 4), step=(1, 1, 1))], M=8, name="mini1")
    if kind == "vacancies":    # cfg2 shape: non-integer spacing/h, 3% vacancies
        return W.lattice_box(128, 12.0, [dict(cells=(8, 8, 8), step=(1, 1, 1))], M=10,
                             n_vacancies=15, eps=1e-6, seed=seed, name="mini2")
    if kind == "yukawa":       # cfg3 shape: Yukawa, impurities with q - 1 charges
        return W.lattice_box(128, 16.0, [dict(cells=(8, 8, 8), step=(1, 1, 1))], family=W.YUKAWA,
                             lam=0.5, M=12, n_impurities=20, q_range=(-0.5, 1.5), eps=1e-7,
                             seed=seed, name="mini3")
    if kind == "hex":          # cfg4 shape: two offset sublattices, steps (1, sqrt3, 1), vacancies
        s3 = float(np.sqrt(3.0))
        return W.lattice_box(256, 24.0, [dict(cells=(8, 4, 8), step=(1.0, s3, 1.0)),
                                         dict(cells=(8, 4, 8), step=(1.0, s3, 1.0),
                                              offset=(0.5, s3 / 2, 0.0))],
                             M=12, n_vacancies=12, eps=1e-7, seed=seed, name="mini4")
    if kind == "mixed":        # cfg5 shape: vacancies + impurities, eps 1e-8
        return W.lattice_box(256, 20.0, [dict(cells=(12, 12, 12), step=(1, 1, 1))], M=12,
                             n_vacancies=10, n_impurities=10, q_range=(0.0, 2.0), eps=1e-8,
                             seed=seed, name="mini5")
    if kind == "clusters":     # reference API geometry with defect clusters (lattice_sum.hpp:297-330):
        # two product clusters (assembled at rank R), a ragged L-shaped one (per site) and an
        # off-grid impurity, in DefectSpec order
        block = [(a, b, 0) for a in (-2, -1) for b in (0, 1)]
        slab = [(a, 2, c) for a in (1, 2, 3) for c in (-1, 0)]
        ragged = [(2, -2, 1), (2, -3, 1), (3, -2, 1)]
        g = W.from_lattice((8, 8, 4), 16, M=10, defects=[
            (block, -1.0, None), (ragged, -1.0, None), (slab, 0.5, None),
            ([(0, 0, 0)], 0.75, (3.0, -2.0, 1.0))], eps=1e-7, name="clusters")
        assert g.n_defects == 1 + 3 + 1 + 1
        return g
    raise ValueError(kind)


def col_rel_linf(a: np.ndarray, b: np.ndarray) -> float:
    """max over columns of ||a_q - b_q||_inf / ||b_q||_inf (directional-vector parity)."""
    den = np.max(np.abs(b), axis=0)
    den[den == 0] = 1.0
    return float(np.max(np.max(np.abs(a - b), axis=0) / den))
