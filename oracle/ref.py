"""TEST INFRASTRUCTURE: ctypes driver for oracle/_ref/liblatsum_ref.so, the reference's own
headers (/root/reference/proj/include/latsum, compiled where they lie by oracle/Makefile against
the Eigen stand-in oracle/shim) behind the small C ABI of oracle/ref_driver.cpp.

This is the reference itself run here, used to pin the CPU restatement (oracle.py /
latsum_oracle.cpp) and the CUDA path to reference OUTPUTS.  `CASES` are geometries the
reference API can express (integral points per cell); `geometry(case)` gives the same case as
the shift-table `Geometry` the oracle port and the CUDA path consume.  Only tests/ and
tests/golden/make_refpin.py import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "liblatsum_ref.so")
UNIT = os.path.join(HERE, "_ref", "ref_unit_tests")
REFERENCE_ROOT = "/root/reference/proj"

_lib = None


def build() -> bool:
    """Compile oracle/_ref from the reference sources when they are present (this container);
    a GPU box only has the prebuilt files.  Returns whether the library exists afterwards."""
    if os.path.isdir(os.path.join(REFERENCE_ROOT, "include", "latsum")):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])
    return os.path.exists(SO)


def available() -> bool:
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise RuntimeError("oracle/_ref/liblatsum_ref.so is not built (make -C oracle ref; "
                               "needs /root/reference)")
        L = C.CDLL(SO)
        L.lref_create.restype = C.c_void_p
        L.lref_last_error.restype = C.c_char_p
        L.lref_last_error.argtypes = [C.c_void_p]
        L.lref_rank_for_tolerance.restype = C.c_int64
        _lib = L
    return _lib


def _p(a, t=C.c_double):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def _ints(x):
    return np.ascontiguousarray(np.asarray(x, np.int32).reshape(-1))


# ----------------------------------------------------------------------------- cases
# Reference-API descriptions: cells, n_per_cell, cell_width, kernel, M, eps, optional active K
# sets, optional sublattices [(cells, offset_cells)] under parent cells, defects
# [(sites, charge, grid_offset | None)].
def _sample_vacancies(cells, count, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    ks = [np.arange(-(c // 2), (c + 1) // 2) for c in cells]
    flat = rng.choice(len(ks[0]) * len(ks[1]) * len(ks[2]), size=count, replace=False)
    out = []
    for f in flat:
        a, r = divmod(int(f), len(ks[1]) * len(ks[2]))
        b, c = divmod(r, len(ks[2]))
        out.append((int(ks[0][a]), int(ks[1][b]), int(ks[2][c])))
    return out


def _cases() -> Dict[str, dict]:
    block = [(a, b, 0) for a in (-2, -1) for b in (0, 1)]
    slab = [(a, 2, c) for a in (1, 2, 3) for c in (-1, 0)]
    ragged = [(2, -2, 1), (2, -3, 1), (3, -2, 1)]
    vac = _sample_vacancies((8, 8, 8), 15, 11)
    imp = _sample_vacancies((8, 8, 8), 12, 12)
    rng = np.random.Generator(np.random.PCG64(13))
    q = rng.uniform(-0.5, 1.5, size=len(imp))
    vac_l = _sample_vacancies((16, 16, 16), 60, 14)
    return {
        # cfg1 shape: cubic, no defects
        "cubic": dict(cells=(4, 4, 4), n=16, b=2.0, family=0, lam=0.0, M=8, eps=1e-6),
        # cfg2 shape: single-site vacancies (one DefectSpec each)
        "vacancies": dict(cells=(8, 8, 8), n=16, b=1.5, family=0, lam=0.0, M=10, eps=1e-6,
                          defects=[([s], -1.0, None) for s in vac]),
        # cfg3 shape: Yukawa, impurities carrying q - 1, one of them off the lattice points
        "yukawa": dict(cells=(8, 8, 8), n=16, b=2.0, family=1, lam=0.5, M=12, eps=1e-7,
                       defects=[([s], float(qq) - 1.0, (3.0, -2.0, 1.0) if i == 0 else None)
                                for i, (s, qq) in enumerate(zip(imp, q))]),
        # cfg4 shape: union of two offset sublattices + vacancies of the first one
        "union": dict(cells=(8, 8, 4), n=16, b=1.0, family=0, lam=0.0, M=10, eps=1e-7,
                      sublattices=[((4, 4, 4), (-1.0, 0.0, 0.0)), ((4, 2, 4), (2.5, 2.5, 0.0))],
                      defects=[([(-1, 0, 1)], -1.0, (-16.0, 0.0, 0.0)),
                               ([(0, -1, -1)], -1.0, (-16.0, 0.0, 0.0))]),
        # defect clusters: two Cartesian products (rank R each), a ragged one (per site), off-grid
        "clusters": dict(cells=(8, 8, 4), n=16, b=1.0, family=0, lam=0.0, M=10, eps=1e-7,
                         defects=[(block, -1.0, None), (ragged, -1.0, None), (slab, 0.5, None),
                                  ([(0, 0, 0)], 0.75, (3.0, -2.0, 1.0))]),
        # a larger cfg2-shaped case (N = 256, M_c = 2013; no canonical_to_tucker: c2t = False)
        "large": dict(cells=(16, 16, 16), n=16, b=1.0, family=0, lam=0.0, M=16, eps=1e-7, c2t=False,
                      defects=[([s], -1.0, None) for s in vac_l]),
        # per-defect kernels (DefectSpec.kernel): a Newton lattice with a Newton vacancy, a Yukawa
        # impurity pair (a product cluster at that kernel's reference rank), another Newton
        # vacancy and a second Yukawa impurity, in this order (add_concat order)
        "mixed_kernels": dict(cells=(6, 6, 4), n=16, b=1.0, family=0, lam=0.0, M=10, eps=1e-7, c2t=False,
                              defects=[([(1, 1, 0)], -1.0, None),
                                       ([(-2, 0, 1), (-1, 0, 1)], 0.6, None, (1, 0.8)),
                                       ([(0, -2, -1)], -1.0, None),
                                       ([(2, 2, 1)], -0.4, (1.0, 0.0, -2.0), (1, 0.8))]),
        # non-contiguous active K sets (the ascending, not sliding, accumulation branch)
        "active": dict(cells=(6, 6, 6), n=12, b=1.0, family=0, lam=0.0, M=8, eps=1e-6,
                       active=[[-3, -2, 0, 1], [-3, -1, 0, 2], [-2, -1, 0, 1, 2]]),
    }


CASES = _cases()


def single_kernel_cases():
    """The cases every defect of which uses the lattice's kernel (one Geometry each)."""
    return [n for n, c in CASES.items()
            if not any(len(d) > 3 and d[3] is not None for d in c.get("defects", ()))]


def geometry_parts(name: str):
    """A case whose defects carry their own kernels, as the add_concat chain defected_sum builds
    (lattice_sum.hpp:355-378): [(family, lambda, Geometry)] — the base lattice with the leading
    base-kernel defects, then one part per maximal run of defects sharing a kernel (geometries
    with no lattice of their own), in DefectSpec order."""
    from paper_1411_1994_b200 import workload as W
    c = CASES[name]
    base_k = (c["family"], c["lam"])
    runs = []  # (kernel, [defects])
    for d in c.get("defects", ()):
        k = tuple(d[3]) if len(d) > 3 and d[3] is not None else base_k
        if runs and runs[-1][0] == k:
            runs[-1][1].append(d[:3])
        else:
            runs.append((k, [d[:3]]))
    parts = []
    lead = runs.pop(0)[1] if runs and runs[0][0] == base_k else []
    parts.append((base_k[0], base_k[1], W.from_lattice(
        c["cells"], c["n"], c["b"], family=base_k[0], lam=base_k[1], M=c["M"], base_charge=1.0,
        active=c.get("active"), defects=lead, eps=c["eps"], name="refpin-" + name)))
    for k, ds in runs:
        parts.append((k[0], k[1], W.from_lattice(
            c["cells"], c["n"], c["b"], family=k[0], lam=k[1], M=c["M"], base_charge=1.0,
            defects=ds, sublattices=[], parent_cells=c["cells"], eps=c["eps"],
            name="refpin-" + name + "-part")))
    return parts


def geometry(name: str):
    """The case as the shift-table Geometry of the oracle port / CUDA path (workload.from_lattice
    applies the reference's own mapping, lattice_sum.hpp:159-164,444)."""
    from paper_1411_1994_b200 import workload as W
    c = CASES[name]
    if any(len(d) > 3 and d[3] is not None for d in c.get("defects", ())):
        raise ValueError("case with per-defect kernels: use geometry_parts")
    return W.from_lattice(c["cells"] if "sublattices" not in c else c["cells"], c["n"], c["b"],
                          family=c["family"], lam=c["lam"], M=c["M"], base_charge=1.0,
                          active=c.get("active"), defects=c.get("defects", ()),
                          sublattices=c.get("sublattices"),
                          parent_cells=c["cells"] if "sublattices" in c else None,
                          eps=c["eps"], name="refpin-" + name)


# ----------------------------------------------------------------------------- driver
class RefRun:
    """One reference run: reference tensor -> canonical sum -> reduction -> entries."""

    def __init__(self, name):
        c = CASES[name] if isinstance(name, str) else dict(name)  # a case name or a case dict
        self.case = c
        L = lib()
        act = c.get("active")
        act_flat = _ints(np.concatenate([np.asarray(a) for a in act])) if act else None
        n_act = _ints([len(a) for a in act]) if act else None
        cells = _ints(c["cells"])
        self.h = L.lref_create(C.c_int(c["family"]), C.c_double(c["lam"]), C.c_int(c["M"]),
                               _p(cells, C.c_int), C.c_int(c["n"]), C.c_double(c["b"]),
                               C.c_double(1.0), C.c_double(0.0), _p(act_flat, C.c_int),
                               _p(n_act, C.c_int))
        if not self.h:
            raise RuntimeError("lref_create: " + L.lref_last_error(None).decode())
        self.h = C.c_void_p(self.h)

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference call failed ({rc}): " + lib().lref_last_error(self.h).decode())

    def close(self):
        if self.h:
            lib().lref_destroy(self.h)
            self.h = None

    def reference(self) -> dict:
        info = np.zeros(7, np.int64)
        c0 = C.c_double()
        shell = np.zeros(2)
        self._check(lib().lref_ref_info(self.h, _p(info, C.c_int64), C.byref(c0), _p(shell)))
        R = int(info[3])
        f = [np.zeros((int(info[l]), R), order="F") for l in range(3)]
        w, t, a = np.zeros(R), np.zeros(R), np.zeros(R)
        self._check(lib().lref_ref_copy(self.h, _p(f[0]), _p(f[1]), _p(f[2]), _p(w), _p(t), _p(a)))
        return dict(factors=f, weights=w, nodes=t, quad_weights=a, C0=c0.value,
                    shell=(float(shell[0]), float(shell[1])), N=tuple(int(x) for x in info[4:7]))

    def _marshal(self):
        c = self.case
        subs = c.get("sublattices") or []
        defs = c.get("defects") or []
        sub_cells = _ints([s[0] for s in subs]) if subs else None
        sub_off = np.ascontiguousarray(np.asarray([s[1] for s in subs], np.float64).reshape(-1)) if subs else None
        nsites = _ints([len(d[0]) for d in defs]) if defs else None
        sites = _ints(np.concatenate([np.asarray(d[0], np.int32).reshape(-1, 3) for d in defs])) if defs else None
        charge = np.ascontiguousarray(np.asarray([d[1] for d in defs], np.float64)) if defs else None
        goff = np.ascontiguousarray(np.asarray([d[2] if d[2] is not None else (0.0, 0.0, 0.0)
                                                for d in defs], np.float64).reshape(-1)) if defs else None
        kind = _ints([0 if d[1] == -1.0 else 1 for d in defs]) if defs else None
        self._keep = (sub_cells, sub_off, nsites, sites, charge, goff, kind)
        return (C.c_int(len(subs)), _p(sub_cells, C.c_int), _p(sub_off), C.c_int(len(defs)),
                _p(nsites, C.c_int), _p(sites, C.c_int), _p(charge), _p(goff), _p(kind, C.c_int))

    def sum(self, accumulation: int = 0):
        """The canonical sum through the library functions (assembled_sum_canonical or
        sublattice_union_sum, then defected_sum).  Defects given as 4-tuples carry their own
        kernel (family, lambda) as DefectSpec.kernel does."""
        defs = self.case.get("defects") or []
        fam = _ints([d[3][0] if len(d) > 3 and d[3] is not None else -1 for d in defs])
        lam = np.ascontiguousarray([d[3][1] if len(d) > 3 and d[3] is not None else 0.0 for d in defs], np.float64)
        self._check(lib().lref_set_defect_kernels(self.h, C.c_int(len(defs)), _p(fam, C.c_int), _p(lam)))
        self._check(lib().lref_sum(self.h, *self._marshal(), C.c_int(accumulation)))
        return self

    def cmd_sum(self, eps: Optional[float] = None, max_als_sweeps: int = -1, seed: int = 0,
                tensor_path=None, provenance_path=None, report_path=None) -> str:
        """The reference's own `latsum sum` (cmd_sum, src/commands.cpp:108-177): with eps the
        result is canonical_to_tucker's.  Sublattice cases ignore defects, as cmd_sum does.
        Returns the command's log."""
        def path(p):
            return C.c_char_p(str(p).encode()) if p else None
        buf = C.create_string_buffer(1 << 16)
        args = list(self._marshal())
        if self.case.get("sublattices"):
            args[3] = C.c_int(0)
        self._check(lib().lref_cmd_sum(self.h, *args, C.c_double(eps or 0.0), C.c_int(max_als_sweeps),
                                       C.c_uint64(seed), path(tensor_path), path(provenance_path),
                                       path(report_path), buf, C.c_int64(1 << 16)))
        return buf.value.decode()

    def cmd_verify(self, tensor_path, provenance_path=None, probes: int = 500,
                   tolerance: float = 1e-10, bound_abs: float = -1.0, seed: int = 0):
        """The reference's own `latsum verify` (cmd_verify, src/commands.cpp:200-284) on a stored
        tensor file -> (ok, log, error)."""
        buf = C.create_string_buffer(1 << 16)
        rc = lib().lref_cmd_verify(self.h, C.c_char_p(str(tensor_path).encode()),
                                   C.c_char_p(str(provenance_path).encode()) if provenance_path else None,
                                   C.c_int(probes), C.c_double(tolerance), C.c_double(bound_abs),
                                   C.c_uint64(seed), buf, C.c_int64(1 << 16))
        return rc == 0, buf.value.decode(), ("" if rc == 0 else lib().lref_last_error(self.h).decode())

    def tucker(self) -> dict:
        """The Tucker result held by the handle (after reduce or a truncated cmd_sum)."""
        return self._tucker()

    def canonical(self):
        rank, ns = C.c_int64(), C.c_int64()
        self._check(lib().lref_canonical_info(self.h, C.byref(rank), C.byref(ns)))
        N = self.reference_dims()
        f = [np.zeros((N[l], rank.value), order="F") for l in range(3)]
        w = np.zeros(rank.value)
        self._check(lib().lref_canonical_copy(self.h, _p(f[0]), _p(f[1]), _p(f[2]), _p(w)))
        return f, w

    def summands(self):
        rank, ns = C.c_int64(), C.c_int64()
        self._check(lib().lref_canonical_info(self.h, C.byref(rank), C.byref(ns)))
        out = []
        for s in range(ns.value):
            buf = C.create_string_buffer(128)
            r, sites = C.c_int64(), C.c_int64()
            self._check(lib().lref_summand(self.h, C.c_int(s), buf, C.c_int(128), C.byref(r), C.byref(sites)))
            out.append((buf.value.decode(), int(r.value), int(sites.value)))
        return out

    def reference_dims(self):
        info = np.zeros(7, np.int64)
        self._check(lib().lref_ref_info(self.h, _p(info, C.c_int64), None, None))
        return tuple(int(x) for x in info[4:7])

    def reduce(self, mode: str = "rhosvd", eps: Optional[float] = None, ranks=None,
               max_als_sweeps: int = -1) -> dict:
        rk = np.asarray(ranks, np.int64) if ranks is not None else None
        self._check(lib().lref_reduce(self.h, C.c_int(0 if mode == "rhosvd" else 1),
                                      C.c_double(eps if eps is not None else 0.0),
                                      _p(rk, C.c_int64), C.c_int(max_als_sweeps)))
        return self._tucker()

    def _tucker(self) -> dict:
        r, nsv, rep, ties = np.zeros(3, np.int64), np.zeros(3, np.int64), np.zeros(6), np.zeros(3, np.int32)
        self._check(lib().lref_tucker_info(self.h, _p(r, C.c_int64), _p(nsv, C.c_int64), _p(rep),
                                           _p(ties, C.c_int)))
        N = self.reference_dims()
        core = np.zeros(tuple(int(x) for x in r), order="F")
        U = [np.zeros((N[l], int(r[l])), order="F") for l in range(3)]
        sv = [np.zeros(int(nsv[l])) for l in range(3)]
        self._check(lib().lref_tucker_copy(self.h, _p(core), _p(U[0]), _p(U[1]), _p(U[2]),
                                           _p(sv[0]), _p(sv[1]), _p(sv[2])))
        return dict(ranks=tuple(int(x) for x in r), sv=sv, core=core, U=U,
                    bound_abs=rep[0], bound_rel=rep[1], weight_norm=rep[2], input_norm=rep[3],
                    stability_constant=rep[4], stability_ok=bool(rep[5]),
                    ties=tuple(bool(t) for t in ties))

    def entries(self, which: str, probes: np.ndarray) -> np.ndarray:
        pr = np.ascontiguousarray(probes, np.int64)
        out = np.zeros(pr.shape[0])
        code = {"canonical": 0, "tucker": 1, "oracle": 2}[which]
        self._check(lib().lref_entries(self.h, C.c_int(code), C.c_int64(pr.shape[0]),
                                       _p(pr, C.c_int64), _p(out)))
        return out


    def _text(self, fn, *args) -> str:
        fn.restype = C.c_int64
        n = fn(self.h, *args, None, C.c_int64(0))
        if n < 0:
            raise RuntimeError("reference writer failed: " + lib().lref_last_error(self.h).decode())
        buf = C.create_string_buffer(int(n) + 1)
        fn(self.h, *args, buf, C.c_int64(n + 1))
        return buf.value.decode()

    def spectral_report_text(self) -> str:
        """write_spectral_report (src/report.cpp:28-47) of the last reduction."""
        return self._text(lib().lref_spectral_report_text)

    def provenance_text(self, seed: int, reduced: bool, extra: str = "") -> str:
        """write_provenance (src/report.cpp:49-73) as cmd_sum records the sum."""
        return self._text(lib().lref_provenance_text, C.c_uint64(seed), C.c_int(int(reduced)),
                          C.c_char_p(extra.encode()))

    def write_tensor(self, which: str, path: str) -> None:
        """write_tensor (src/tensor_io.cpp) of the canonical sum or the Tucker result."""
        self._check(lib().lref_write_tensor(self.h, C.c_int(0 if which == "canonical" else 1),
                                            C.c_char_p(str(path).encode())))


def read_tensor_entries(path, probes):
    """read_tensor (src/tensor_io.cpp) + entries at the probes -> (kind, dims, values); raises
    IOError on the reference's TensorIoError."""
    pr = np.ascontiguousarray(probes, np.int64)
    out = np.zeros(pr.shape[0])
    kind = C.c_int()
    dims = np.zeros(3, np.int64)
    rc = lib().lref_read_tensor_entries(C.c_char_p(str(path).encode()), C.byref(kind),
                                        _p(dims, C.c_int64), C.c_int64(pr.shape[0]),
                                        _p(pr, C.c_int64), _p(out))
    if rc == 5:
        raise IOError(lib().lref_last_error(None).decode())
    if rc != 0:
        raise RuntimeError(lib().lref_last_error(None).decode())
    return ("canonical", "tucker")[kind.value], tuple(int(x) for x in dims), out


def assembled_vector(ref_col, kset, n, off, nl, accumulation=0):
    ref_col = np.ascontiguousarray(ref_col, np.float64)
    ks = _ints(kset)
    out = np.zeros(nl)
    rc = lib().lref_assembled_vector(_p(ref_col), C.c_int64(ref_col.size), _p(ks, C.c_int),
                                     C.c_int(ks.size), C.c_int64(n), C.c_long(off), C.c_int64(nl),
                                     C.c_int(accumulation), _p(out))
    if rc != 0:
        raise RuntimeError(f"assembled_vector failed ({rc}): " + lib().lref_last_error(None).decode())
    return out


def rank_for_tolerance(sv, eps) -> int:
    sv = np.ascontiguousarray(sv, np.float64)
    return int(lib().lref_rank_for_tolerance(_p(sv), C.c_int64(sv.size), C.c_double(eps)))


def quadrature(family, lam, M, C0, a, A):
    R = 2 * M + 1
    t, w = np.zeros(R), np.zeros(R)
    c0 = C.c_double()
    rc = lib().lref_quadrature(C.c_int(family), C.c_double(lam), C.c_int(M), C.c_double(C0),
                               C.c_double(a), C.c_double(A), C.byref(c0), _p(t), _p(w))
    if rc != 0:
        raise RuntimeError(f"quadrature failed ({rc}): " + lib().lref_last_error(None).decode())
    return c0.value, t, w


def run_unit_tests() -> str:
    """The reference's own unit tests (tests/unit/*.cpp minus the JSON/config ones), compiled
    against the stand-ins; returns the summary line."""
    out = subprocess.run([UNIT], capture_output=True, text=True, timeout=600)
    return out.stdout.strip().splitlines()[-1] + f" | rc={out.returncode}"
