"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/latsum_b200.h declares, and the host-side rules are callable."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1411_1994_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "latsum_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(latsum_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(ValueError):
        _lib.check(1)
    with pytest.raises(IndexError):
        _lib.check(2)
    with pytest.raises(OverflowError):
        _lib.check(6)
    with pytest.raises(NotImplementedError):
        _lib.check(7)


def test_host_quadrature_rejects_bad_rules():
    L = _lib.lib()
    t, a = np.zeros(3), np.zeros(3)
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    assert L.latsum_build_quadrature(0, 0.0, 1, 1.0, 0.1, 1.0, p(t), p(a)) == 1  # M < 2
    assert L.latsum_build_quadrature(0, 0.0, 2, 1.0, 1.0, 0.5, p(t), p(a)) == 1  # a >= A
    assert L.latsum_build_quadrature(3, 0.0, 2, 1.0, 0.1, 1.0, p(t), p(a)) == 7  # slater: not on path


def test_context_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_1411_1994_b200 import api
    with pytest.raises(RuntimeError):
        api.Context(0)


def test_host_step_constant_matches_oracle_across_threads():
    """quadrature.hpp:238-269 (default_step_constant) in the library — evaluated on its
    persistent host worker pool — equals the oracle's sequential sweep bit for bit, for the
    five BASELINE configurations, also when several host threads call it at once."""
    import threading

    from oracle import oracle as O
    from paper_1411_1994_b200 import workload as W

    L = _lib.lib()
    cases = []
    for cfg in range(1, 6):
        g = W.baseline(cfg)
        a, A = O.reference_shell(g.N, g.box)
        cases.append((g.family, g.lam, g.M, a, A, O.default_step_constant(g.family, g.lam, g.M, a, A)))
    got = {}

    def run(tid):
        for i, (fam, lam, M, a, A, _) in enumerate(cases):
            got[(tid, i)] = L.latsum_default_step_constant(fam, lam, M, a, A, 320)

    threads = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for (tid, i), c0 in got.items():
        assert c0 == cases[i][5], (tid, i, c0, cases[i][5])
