"""Generates the golden fixtures in this directory (run here, where mpmath exists):

  cell_integrals.json  50-digit integrals of exp(-s x^2) over double-valued cells
                       [lo, lo + h] of the BASELINE doubled grids (reference.hpp:33-54)
  quadrature.json      40-digit sinc nodes/weights (quadrature.hpp:155-163) evaluated
                       from the same double-valued step and abscissae the code forms,
                       plus the calibrated C0 and an independent 4-digit C0 probe value
                       (SURVEY 8a row a2).

    python tests/golden/make_golden.py
"""
import json
import math
import os
import sys

import mpmath as mp
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1411_1994_b200 import workload as W  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
C0_PROBE = {1: 2.9529, 2: 3.1841, 3: 2.3076, 4: 3.3520, 5: 3.6229}


def cell_integral(s, lo, h):
    mp.mp.dps = 60
    s_, lo_ = mp.mpf(s), mp.mpf(lo)
    hi_ = mp.mpf(lo + h)  # the code's hi = lo + h, rounded to double
    rs = mp.sqrt(s_)
    return mp.sqrt(mp.pi) / (2 * rs) * (mp.erf(rs * hi_) - mp.erf(rs * lo_))


def main():
    cells, quad = [], []
    rng = np.random.default_rng(1994)
    for cfg in range(1, 6):
        g = W.baseline(cfg)
        a, A = O.reference_shell(g.N, g.box)
        c0 = O.default_step_constant(g.family, g.lam, g.M, a, A)
        t, w = O.quadrature(g.family, g.lam, g.M, c0, a, A)
        # golden nodes / weights from the double-valued step and abscissae
        mp.mp.dps = 40
        hM = c0 * math.log(float(g.M)) / float(g.M)
        gn, gw = [], []
        for k in range(2 * g.M + 1):
            u = (float(k) - float(g.M)) * hM
            tk = mp.sinh(mp.mpf(u)) / mp.mpf(A)
            td = float(tk)
            if g.family == W.NEWTON:
                wt = mp.mpf(2.0 / math.sqrt(math.pi))
            else:
                kap = g.lam / 2.0
                wt = mp.mpf(0.0) if td == 0.0 else mp.mpf(2.0 / math.sqrt(math.pi)) * mp.exp(
                    mp.mpf(-(kap * kap) / (abs(td) * abs(td))))
            ak = mp.mpf(0.5 * hM) * wt * mp.cosh(mp.mpf(u)) / mp.mpf(A)
            gn.append(mp.nstr(tk, 30))
            gw.append(mp.nstr(ak, 30))
        quad.append(dict(cfg=cfg, C0=c0, C0_probe=C0_PROBE[cfg], nodes=gn, weights=gw))
        # cells of three columns: sharpest, middle, widest nonzero
        n2 = 2 * g.N[0]
        h = (2.0 * g.box[0]) / float(n2)
        lower = 0.0 - (2.0 * g.box[0]) / 2.0
        for k in (0, g.M // 2, g.M - 1):
            s = t[k] * t[k]
            col = O.mode_integrals(np.array([t[k]]), n2, lower, h, "hybrid")[:, 0]
            colmax = float(np.max(np.abs(col)))
            idx = {0, 1, n2 // 4 - 1, n2 // 4, n2 // 2 - 2, n2 // 2 - 1, n2 // 2, n2 // 2 + 1,
                   3 * n2 // 4, n2 - 1}
            idx |= set(int(x) for x in rng.integers(0, n2, 6))
            idx |= set(int(x) for x in rng.integers(n2 // 2 - 64, n2 // 2 + 64, 6))
            for i in sorted(idx):
                lo = lower + float(i) * h
                v = cell_integral(s, lo, h)
                cells.append(dict(cfg=cfg, k=k, i=i, s=s, lo=lo, h=h, value=mp.nstr(v, 30),
                                  colmax=colmax))
    json.dump(dict(cells=cells), open(os.path.join(HERE, "cell_integrals.json"), "w"), indent=0)
    json.dump(dict(configs=quad), open(os.path.join(HERE, "quadrature.json"), "w"), indent=0)
    print(len(cells), "cells;", [q["C0"] for q in quad])


if __name__ == "__main__":
    main()
