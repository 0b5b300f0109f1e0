"""Lattice geometries in grid (shift-table) form, and the BASELINE workloads.

The reference describes a lattice by `LatticeGeometry` (cells, cell width,
active K sets, `DefectSpec` sites with `grid_offset`, sublattice offsets) and
maps it to integer mesh shifts in two places:

* base sources: ``c = k * n_per_cell + lround(offset_cells * n_per_cell)``
  (``lattice_sum.hpp:444`` sublattice_union_sum, ``:632-641`` enumerate_sources);
* defect sites: ``c = site * n_per_cell + lround(grid_offset)``
  (``lattice_sum.hpp:159-164`` defect_grid_shift).

`from_lattice` reproduces exactly that mapping.  The BASELINE configs 2-5 put a
lattice whose spacing is not a whole number of mesh cells into a box larger
than the lattice, which the reference cannot express; `cubic` and
`baseline` therefore snap every site position to the grid with the
reference's own rule (``grid.hpp:120-135`` snap_to_grid: round half away from
zero) and keep the lattice rank-preserving per mode because the site set is
still a tensor product per sublattice.

A `Geometry` is the one exchange format shared by the CUDA path and the CPU
oracle: per-sublattice per-mode shift lists, and per-defect shift triples with
additive charges (vacancy = -base charge, impurity = q - base charge,
``config.cpp:105-110``, ``lattice_sum.hpp:306``).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

NEWTON = 0
YUKAWA = 1


@dataclass
class Sublattice:
    shifts: Tuple[np.ndarray, np.ndarray, np.ndarray]  # per-mode int64 mesh shifts, K order
    charge: float = 1.0


@dataclass
class Geometry:
    N: Tuple[int, int, int]
    box: Tuple[float, float, float]  # full box widths b_l; mesh h_l = b_l / N_l
    family: int = NEWTON
    lam: float = 0.0
    M: int = 16
    C0: float = 0.0  # <= 0: calibrated sweep (quadrature.hpp:238-269)
    sublattices: List[Sublattice] = field(default_factory=list)
    defect_shifts: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int64))
    defect_charges: np.ndarray = field(default_factory=lambda: np.zeros((0,), np.float64))
    # Defects in DefectSpec order as product blocks (lattice_sum.hpp:297-330): a cluster
    # whose sites form a Cartesian product is ONE block at reference rank
    # (product_structure), any other cluster one 1 x 1 x 1 block per site.  None: every
    # defect is the single site of the matching defect_shifts row.
    defect_blocks: Optional[List[Sublattice]] = None
    eps: Optional[float] = None  # RHOSVD tolerance (None: no truncation)
    eval_lo: Tuple[int, int, int] = (0, 0, 0)
    eval_hi: Optional[Tuple[int, int, int]] = None
    name: str = ""
    seed: int = 0
    n_vacancies: int = 0   # sampled defects by kind (lattice_box); informational
    n_impurities: int = 0
    # provenance (lattice_sum.hpp:44-50 Summand): (label, canonical rank, sites) per
    # summand, and the geometry's cell counts; None: derived (summands())
    summand_list: Optional[List[Tuple[str, int, int]]] = None
    cells: Optional[Tuple[int, int, int]] = None

    @property
    def R(self) -> int:
        return 2 * self.M + 1

    @property
    def h(self) -> Tuple[float, float, float]:
        return tuple(float(b) / float(n) for b, n in zip(self.box, self.N))

    @property
    def n_defects(self) -> int:
        """Defect blocks: product clusters count once, other sites one each."""
        if self.defect_blocks is not None:
            return len(self.defect_blocks)
        return int(self.defect_shifts.shape[0])

    @property
    def canonical_rank(self) -> int:
        """M_c = R * (#sublattices + #defect blocks): rank of the unreduced sum."""
        return self.R * (len(self.sublattices) + self.n_defects)

    def summands(self) -> List[Tuple[str, int, int]]:
        """The summands a LatticeSumResult records (commands.cpp:157-163,
        lattice_sum.hpp:368-370, :453-454): the assembled lattice sum (or one per
        sublattice), then one vacancy / impurity cluster per defect."""
        if self.summand_list is not None:
            return list(self.summand_list)
        out = []
        for sub in self.sublattices:
            sites = int(np.prod([len(x) for x in sub.shifts]))
            out.append(("assembled lattice sum" if len(self.sublattices) == 1 else "sublattice",
                         self.R, sites))
        for b in self.blocks()[len(self.sublattices):]:
            sites = int(np.prod([len(x) for x in b.shifts]))
            out.append(("vacancy cluster" if b.charge < 0 else "impurity cluster", self.R, sites))
        return out

    def cell_counts(self) -> Tuple[int, int, int]:
        if self.cells is not None:
            return tuple(int(x) for x in self.cells)
        if self.sublattices:
            return tuple(len(x) for x in self.sublattices[0].shifts)
        return (0, 0, 0)

    def blocks(self) -> List[Sublattice]:
        """Every product block in add_concat order: the sublattices, then the defects."""
        out = list(self.sublattices)
        if self.defect_blocks is not None:
            out += list(self.defect_blocks)
        else:
            out += [Sublattice(tuple(np.array([s[l]], np.int64) for l in range(3)), float(q))
                    for s, q in zip(self.defect_shifts, self.defect_charges)]
        return out

    @property
    def n_sites(self) -> int:
        return int(sum(np.prod([len(s) for s in sub.shifts]) for sub in self.sublattices))

    def eval_box(self):
        hi = self.eval_hi if self.eval_hi is not None else self.N
        return tuple(self.eval_lo), tuple(hi)

    def sources(self):
        """All grid-shifted sources (lattice_sum.hpp:632-653 enumerate_sources): base
        sites of every sublattice (charge = sublattice charge), then every defect."""
        shifts, weights = [], []
        for sub in self.sublattices:
            a, b, c = np.meshgrid(sub.shifts[0], sub.shifts[1], sub.shifts[2], indexing="ij")
            # active_cells order: ascending (k3, k2, k1), k1 fastest
            s = np.stack([a.transpose(2, 1, 0).ravel(), b.transpose(2, 1, 0).ravel(),
                          c.transpose(2, 1, 0).ravel()], axis=1)
            shifts.append(s)
            weights.append(np.full(s.shape[0], sub.charge))
        if self.defect_shifts.shape[0]:
            shifts.append(self.defect_shifts)
            weights.append(self.defect_charges)
        return (np.ascontiguousarray(np.concatenate(shifts).astype(np.int64)),
                np.ascontiguousarray(np.concatenate(weights).astype(np.float64)))


def default_active_set(cells: int) -> np.ndarray:
    """geometry.hpp:36-40: K = {-floor(L/2), ..., ceil(L/2)-1}."""
    return np.arange(-(cells // 2), (cells + 1) // 2, dtype=np.int64)


def snap(x: np.ndarray, h: float) -> np.ndarray:
    """grid.hpp:131: std::round (half away from zero) of x/h."""
    q = np.asarray(x, dtype=np.float64) / h
    return (np.sign(q) * np.floor(np.abs(q) + 0.5)).astype(np.int64)


def lround(x: float) -> int:
    """std::lround: round half away from zero."""
    return int(np.sign(x) * np.floor(abs(x) + 0.5))


def product_structure(sites: Sequence[Sequence[int]]):
    """lattice_sum.hpp:278-294: the per-mode sorted index sets if the sites form their
    full Cartesian product (every combination present, none repeated), else None."""
    axes = [sorted({int(s[l]) for s in sites}) for l in range(3)]
    if len(axes[0]) * len(axes[1]) * len(axes[2]) != len(sites):
        return None
    have = {tuple(int(v) for v in s) for s in sites}
    for a in axes[0]:
        for b in axes[1]:
            for c in axes[2]:
                if (a, b, c) not in have:
                    return None
    return axes


def from_lattice(cells: Sequence[int], n_per_cell: int, cell_width: float = 1.0, *,
                 family: int = NEWTON, lam: float = 0.0, M: int = 8, C0: float = 0.0,
                 base_charge: float = 1.0, active: Optional[Sequence[Sequence[int]]] = None,
                 defects: Sequence[Tuple[Sequence[Sequence[int]], float, Sequence[float]]] = (),
                 sublattices: Optional[Sequence[Tuple[Sequence[int], Sequence[float]]]] = None,
                 parent_cells: Optional[Sequence[int]] = None,
                 eps: Optional[float] = None, name: str = "") -> Geometry:
    """Reference-API geometry -> shift tables.

    lattice_grid (lattice_sum.hpp:75-86): N_l = n * L_l, box_l = b * L_l.
    Base shifts c = k n (assembled_sum_canonical, :198-223); sublattice shifts
    c = k n + lround(offset n) (:444); defect shifts c = site n + lround(grid_offset)
    (:159-164).  `defects` entries are (sites, charge, grid_offset): a cluster whose
    sites form a Cartesian product is one R-term block over the per-mode sorted index sets
    (product_structure, :316-321); any other cluster contributes one R-term block per site
    in site order (:324-329).
    """
    grid_cells = list(parent_cells) if parent_cells is not None else list(cells)
    N = tuple(int(n_per_cell * c) for c in grid_cells)
    box = tuple(float(cell_width) * float(c) for c in grid_cells)
    subs: List[Sublattice] = []
    if sublattices is None:
        ks = [np.asarray(active[l], np.int64) if active is not None and len(active[l])
              else default_active_set(cells[l]) for l in range(3)]
        ks = [np.sort(k) for k in ks]  # assembled_vector sorts the K set
        subs.append(Sublattice(tuple(k * n_per_cell for k in ks), base_charge))
    else:
        for sub_cells, off in sublattices:
            ks = [default_active_set(sub_cells[l]) for l in range(3)]
            subs.append(Sublattice(tuple(ks[l] * n_per_cell + lround(off[l] * n_per_cell)
                                         for l in range(3)), base_charge))
    summ = ([("assembled lattice sum", 2 * M + 1, int(np.prod([len(x) for x in subs[0].shifts])))]
            if sublattices is None else
            [("sublattice", 2 * M + 1, int(np.prod([len(x) for x in s.shifts]))) for s in subs])
    dsh, dch, dblk = [], [], []
    for sites, charge, goff in defects:
        goff = goff if goff is not None else (0.0, 0.0, 0.0)
        if not len(sites):
            raise ValueError("defected_sum: defect with no sites")
        off = [lround(goff[l]) for l in range(3)]
        for s in sites:
            dsh.append([int(s[l]) * n_per_cell + off[l] for l in range(3)])
            dch.append(float(charge))
        axes = product_structure(sites) if len(sites) > 1 else None
        # config.cpp:105-110: a vacancy carries -base_charge; anything else is an impurity
        kind = "vacancy cluster" if float(charge) == -float(base_charge) else "impurity cluster"
        summ.append((kind, (2 * M + 1) * (1 if axes is not None or len(sites) == 1 else len(sites)),
                     len(sites)))
        if axes is not None:  # assembled cluster: rank stays at the reference rank
            dblk.append(Sublattice(tuple(np.asarray(axes[l], np.int64) * n_per_cell + off[l]
                                         for l in range(3)), float(charge)))
        else:
            dblk += [Sublattice(tuple(np.array([int(s[l]) * n_per_cell + off[l]], np.int64)
                                      for l in range(3)), float(charge)) for s in sites]
    return Geometry(N=N, box=box, family=family, lam=lam, M=M, C0=C0, sublattices=subs,
                    defect_shifts=np.asarray(dsh, np.int64).reshape(-1, 3),
                    defect_charges=np.asarray(dch, np.float64),
                    defect_blocks=dblk if len(dblk) != len(dsh) else None, eps=eps, name=name,
                    summand_list=summ, cells=tuple(int(c) for c in grid_cells))


def _sample_sites(n_sites: int, count: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.choice(n_sites, size=count, replace=False)


def lattice_box(N: int, box: float, sublats: Sequence[dict], *, family=NEWTON, lam=0.0, M=16,
                n_vacancies=0, n_impurities=0, q_range=(0.0, 2.0), eps=None,
                seed=0x14111994, name="", eval_lo=(0, 0, 0), eval_hi=None) -> Geometry:
    """Generalised cubic-grid geometry (SURVEY F2 / section 8d site convention).

    Each sublattice dict: {"cells": (L1,L2,L3), "step": (a1,a2,a3), "offset": (o1,o2,o3)}:
    sites x_l = k a_l + o_l for k in the reference K set, snapped to the grid.
    Defects: `n_vacancies + n_impurities` distinct sites drawn from the linear
    site index i1 + L1 (i2 + L2 i3) (+ sublattice * L1 L2 L3); the first
    `n_vacancies` drawn are vacancies (charge -1), the rest impurities with
    q ~ U[q_range] and correction charge q - 1.  Defects are ordered by
    ascending site index, which is the canonical column order.
    """
    h = float(box) / float(N)
    subs, per_sub = [], []
    for sd in sublats:
        cells, step, off = sd["cells"], sd["step"], sd.get("offset", (0.0, 0.0, 0.0))
        sh = tuple(snap(default_active_set(cells[l]) * float(step[l]) + float(off[l]), h)
                   for l in range(3))
        for l in range(3):
            if np.any(np.abs(sh[l]) > N // 2):
                raise ValueError(f"lattice does not fit the box in mode {l + 1}")
        subs.append(Sublattice(sh, 1.0))
        per_sub.append(int(np.prod(cells)))
    total = int(sum(per_sub))
    nd = n_vacancies + n_impurities
    dsh = np.zeros((0, 3), np.int64)
    dch = np.zeros((0,), np.float64)
    if nd:
        rng = np.random.Generator(np.random.PCG64(seed))
        drawn = rng.choice(total, size=nd, replace=False)
        charges = np.full(nd, -1.0)
        if n_impurities:
            q = rng.uniform(q_range[0], q_range[1], size=n_impurities)
            charges[n_vacancies:] = q - 1.0
        order = np.argsort(drawn, kind="stable")
        drawn, charges = drawn[order], charges[order]
        kinds = ["vacancy cluster" if o < n_vacancies else "impurity cluster" for o in order]
        rows = []
        starts = np.cumsum([0] + per_sub)
        for idx in drawn:
            s = int(np.searchsorted(starts, idx, side="right") - 1)
            loc = int(idx - starts[s])
            cells = sublats[s]["cells"]
            i1 = loc % cells[0]
            i2 = (loc // cells[0]) % cells[1]
            i3 = loc // (cells[0] * cells[1])
            rows.append([subs[s].shifts[0][i1], subs[s].shifts[1][i2], subs[s].shifts[2][i3]])
        dsh = np.asarray(rows, np.int64).reshape(-1, 3)
        dch = charges.astype(np.float64)
    R = 2 * M + 1
    summ = ([("assembled lattice sum", R, per_sub[0])] if len(subs) == 1 else
            [("sublattice", R, p) for p in per_sub])
    if nd:
        summ += [(k, R, 1) for k in kinds]
    return Geometry(N=(N, N, N), box=(box, box, box), family=family, lam=lam, M=M,
                    summand_list=summ, cells=tuple(int(c) for c in sublats[0]["cells"]),
                    sublattices=subs, defect_shifts=dsh, defect_charges=dch, eps=eps,
                    name=name, seed=seed, eval_lo=tuple(eval_lo), eval_hi=eval_hi,
                    n_vacancies=int(n_vacancies), n_impurities=int(n_impurities))


def baseline(i: int, seed: Optional[int] = None) -> Geometry:
    """BASELINE.json configs[i-1] (i = 1..5) as synthetic seeded geometries."""
    sd = 0x14111994 + i if seed is None else seed
    if i == 1:
        # cubic L=8, spacing 1, box [-8,8]^3, N=512 (h=1/32, stride 32)
        return lattice_box(512, 16.0, [dict(cells=(8, 8, 8), step=(1, 1, 1))], M=16,
                           seed=sd, name="cfg1")
    if i == 2:
        return lattice_box(2048, 48.0, [dict(cells=(32, 32, 32), step=(1, 1, 1))], M=20,
                           n_vacancies=round(0.03 * 32 ** 3), eps=1e-6, seed=sd, name="cfg2")
    if i == 3:
        c = 4096 // 2
        return lattice_box(4096, 80.0, [dict(cells=(64, 64, 64), step=(1, 1, 1))],
                           family=YUKAWA, lam=0.5, M=24, n_impurities=256,
                           q_range=(-0.5, 1.5), eps=1e-7, seed=sd, name="cfg3",
                           eval_lo=(c - 1024,) * 3, eval_hi=(c + 1024,) * 3)
    if i == 4:
        s3 = float(np.sqrt(3.0))
        c = 8192 // 2
        return lattice_box(8192, 144.0, [dict(cells=(96, 48, 96), step=(1.0, s3, 1.0)),
                                         dict(cells=(96, 48, 96), step=(1.0, s3, 1.0),
                                              offset=(0.5, s3 / 2.0, 0.0))],
                           M=28, n_vacancies=500, eps=1e-7, seed=sd, name="cfg4",
                           eval_lo=(c - 1024,) * 3, eval_hi=(c + 1024,) * 3)
    if i == 5:
        c = 32768 // 2
        return lattice_box(32768, 320.0, [dict(cells=(256, 256, 256), step=(1, 1, 1))], M=32,
                           n_vacancies=500, n_impurities=500, q_range=(0.0, 2.0), eps=1e-8,
                           seed=sd, name="cfg5", eval_lo=(c - 1024,) * 3,
                           eval_hi=(c + 1024,) * 3)
    raise ValueError("baseline config index is 1..5")


def row_block(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows [lo, hi) of an n-row operand owned by `rank` (latsum_capi.cu row_block)."""
    return n * rank // world, n * (rank + 1) // world


def z_slab(lo: Sequence[int], hi: Sequence[int], rank: int, world: int):
    """The z-slab of the evaluation box [lo, hi) that `rank` evaluates (no communication)."""
    z0, z1 = row_block(hi[2] - lo[2], rank, world)
    return (lo[0], lo[1], lo[2] + z0), (hi[0], hi[1], lo[2] + z1)


def describe(g: Geometry) -> dict:
    """The workload as one JSON-able dict (bench.py prints it on both arms)."""
    lo, hi = g.eval_box()
    return {
        "workload": g.name,
        "kernel": "yukawa" if g.family == YUKAWA else "newton",
        "lambda": g.lam if g.family == YUKAWA else None,
        "N": int(g.N[0]), "box": float(g.box[0]), "M": int(g.M), "R": int(g.R),
        "sublattices": len(g.sublattices), "sites": int(g.n_sites),
        "vacancies": int(g.n_vacancies), "impurities": int(g.n_impurities),
        "canonical_rank": int(g.canonical_rank), "eps": g.eps, "seed": int(g.seed),
        "eval_box": [list(map(int, lo)), list(map(int, hi))],
    }
