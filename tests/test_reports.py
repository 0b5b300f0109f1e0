"""Spectral report and provenance sidecar (report.cpp:28-73, commands.cpp:56-72): the
library's writers (host-only C ABI) against the oracle's restatement, byte for byte."""
import numpy as np

from oracle import oracle as O
from paper_1411_1994_b200 import api
from paper_1411_1994_b200 import workload as W


def _report(seed=3):
    rng = np.random.default_rng(seed)
    sv = [np.sort(np.abs(rng.standard_normal(n)) * 10.0 ** rng.uniform(-14, 2, n))[::-1]
          for n in (7, 1, 12)]
    sv[1][:] = [0.0]
    return api.SpectralReport(
        singular_values=sv, chosen_ranks=(3, 1, 5), bound_abs=1.2345678901234567e-9,
        bound_rel=float(np.nextafter(1e-7, 1)), weight_norm=123.0, input_norm=1.0 / 3.0,
        stability_constant=4e300, stability_ok=False, tie_at_cutoff=(False, True, False),
        cutoff_margin=(0.1, 0.2, 0.3), deflated=(True, True, True),
        gram_rows=(False, False, False), gram_size=(7, 1, 12), ms={})


def test_spectral_report_matches_reference_writer():
    r = _report()
    got = api.format_spectral_report(r)
    want = O.spectral_report_text(r.chosen_ranks, r.bound_abs, r.bound_rel, r.weight_norm,
                                  r.input_norm, r.stability_constant, r.stability_ok,
                                  r.tie_at_cutoff, r.singular_values)
    assert got == want
    assert "sigma_mode2 (tie at cutoff) 0\n" in got
    assert "stability_constant 4.0000000000000002e+300\n" in got  # 17 significant digits


class _Canonical:  # stands in for a device CanonicalTensor (rank only)
    rank = 187


def test_provenance_matches_reference_writer(tmp_path):
    g = W.from_lattice((8, 8, 1), 8, M=8, defects=[
        ([(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0)], -1.0, None),
        ([(2, 2, 0), (2, 3, 0), (3, 2, 0)], 0.5, None)])
    assert g.summands() == [("assembled lattice sum", 17, 64), ("vacancy cluster", 17, 4),
                            ("impurity cluster", 51, 3)]
    got = api.format_provenance(g, _Canonical(), seed=2 ** 64 - 1, extra_lines=["note x"])
    want = O.provenance_text(2 ** 64 - 1, g.N, (8, 8, 1), "canonical", 187, g.summands(),
                             extra_lines=["note x"])
    assert got == want
    r = _report()
    p = tmp_path / "prov.txt"
    api.write_provenance(str(p), g, _Canonical(), r, seed=7)
    assert p.read_text() == O.provenance_text(7, g.N, (8, 8, 1), "canonical", 187, g.summands(),
                                              bounds=(r.bound_abs, r.bound_rel))


def test_baseline_summands_record_every_defect():
    g = W.baseline(5)
    s = g.summands()
    assert s[0] == ("assembled lattice sum", 65, 256 ** 3)
    assert sum(1 for x in s if x[0] == "vacancy cluster") == 500
    assert sum(1 for x in s if x[0] == "impurity cluster") == 500
    assert g.cell_counts() == (256, 256, 256)
