"""Every `file.hpp:a-b` / `file.cpp:a` citation of the reference in the repo points inside
the cited file (the oracle and the boundary must cite what they restate).

The reference tree is not on the GPU box, so the file lengths are pinned here and
re-checked against /root/reference when it is present (this container)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"

# physical line counts of the reference files (wc -l)
REF_LINES = {
    "cache.hpp": 29, "canonical.hpp": 204, "commands.hpp": 58, "config.hpp": 56,
    "geometry.hpp": 121, "grid.hpp": 137, "kernel.hpp": 178, "lattice_sum.hpp": 702,
    "linalg.hpp": 81, "parallel.hpp": 34, "quadrature.hpp": 332, "rank_reduction.hpp": 476,
    "reference.hpp": 178, "report.hpp": 29, "tensor3.hpp": 107, "tensor_io.hpp": 37,
    "tucker.hpp": 180, "types.hpp": 24, "cache.cpp": 110, "commands.cpp": 352,
    "config.cpp": 276, "report.cpp": 119, "tensor_io.cpp": 131, "acceptance_main.cpp": 544,
    "test_grid_geometry.cpp": 156, "test_helpers.hpp": 94, "test_io_config.cpp": 205,
    "test_kernel_quadrature.cpp": 155, "test_lattice_sum.cpp": 611,
    "test_rank_reduction.cpp": 244, "test_reference.cpp": 192, "test_tensor_formats.cpp": 248,
    "latsum_cli.cpp": 196,
}

# definition lines of functions the code cites by name: a citation on the same line as
# the name must cover the definition
DEFINITIONS = {
    "build_quadrature": ("quadrature.hpp", 125),
    "default_step_constant": ("quadrature.hpp", 238),
    "gauss_weight": ("quadrature.hpp", 73),
    "mode_integrals": ("reference.hpp", 33),
    "reference_shell": ("reference.hpp", 84),
    "snap_to_grid": ("grid.hpp", 121),
    "window_indices": ("grid.hpp", 104),
    "product_structure": ("lattice_sum.hpp", 278),
    "rank_for_tolerance": ("rank_reduction.hpp", 73),
    "project_core": ("rank_reduction.hpp", 88),
    "WindowOverflowError": ("grid.hpp", 87),
    "shrink_core": ("rank_reduction.hpp", 130),
    "write_spectral_report": ("report.cpp", 28),
    "write_provenance": ("report.cpp", 48),
}

# review / survey documents quote the reference as found; they are not citations we own
SKIP = {"VERDICT.md", "ADVICE.md", "SURVEY.md", "BASELINE.md", "PAPERS.md", "SNIPPETS.md",
        "tests/test_citations.py"}
PAT = re.compile(r"([A-Za-z_0-9]+\.(?:hpp|cpp)):(\d+)(?:-(\d+))?((?:,\d+(?:-\d+)?)*)")


def _tracked():
    try:
        out = subprocess.check_output(["git", "ls-files"], cwd=ROOT, text=True,
                                      stderr=subprocess.DEVNULL)
        files = out.split()
    except Exception:  # not a git checkout (e.g. a copied tree)
        files = []
        for d, _, fs in os.walk(ROOT):
            if "/." in d or "gpurun_out" in d:
                continue
            files += [os.path.relpath(os.path.join(d, f), ROOT) for f in fs]
    return [f for f in files if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", ".hpp", ".md"))
            and f not in SKIP]


def _citations():
    for f in _tracked():
        try:
            text = open(os.path.join(ROOT, f), errors="ignore").read()
        except OSError:
            continue
        for i, line in enumerate(text.splitlines(), 1):
            for m in PAT.finditer(line):
                if m.group(1) not in REF_LINES:
                    continue
                ranges = [(int(m.group(2)), int(m.group(3) or m.group(2)))]
                for extra in (m.group(4) or "").split(","):
                    if extra:
                        a, _, b = extra.partition("-")
                        ranges.append((int(a), int(b or a)))
                yield f, i, line, m.group(1), ranges


def test_reference_line_table_matches_tree():
    if not os.path.isdir(REF):
        pytest.skip("reference tree not present (GPU box)")
    seen = {}
    for d, _, fs in os.walk(REF):
        for name in fs:
            if name in REF_LINES:
                seen[name] = sum(1 for _ in open(os.path.join(d, name), errors="ignore"))
    assert seen == REF_LINES


def test_every_citation_is_inside_its_file():
    bad = [(f, i, name, ranges) for f, i, _, name, ranges in _citations()
           if any(a < 1 or b > REF_LINES[name] or b < a for a, b in ranges)]
    assert not bad, bad
    assert sum(1 for _ in _citations()) > 100  # the scan sees the code's citations


def test_named_citations_cover_the_definition():
    """A citation right after a defined function's name (`name` (file.hpp:a-b), name
    file.hpp:a-b, ...) covers that function's definition line."""
    bad = []
    names = "|".join(DEFINITIONS)
    near = re.compile(r"\b(" + names + r")\b[`\s(,:]{0,6}(?:\(`?)?([A-Za-z_0-9]+\.(?:hpp|cpp)):(\d+)(?:-(\d+))?")
    for f in _tracked():
        try:
            text = open(os.path.join(ROOT, f), errors="ignore").read()
        except OSError:
            continue
        for i, line in enumerate(text.splitlines(), 1):
            for m in near.finditer(line):
                fn, file, a, b = m.group(1), m.group(2), int(m.group(3)), int(m.group(4) or m.group(3))
                want_file, defline = DEFINITIONS[fn]
                if file == want_file and not a <= defline <= b:
                    bad.append((f, i, fn, (a, b)))
    assert not bad, bad
