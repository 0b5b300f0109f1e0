"""Reference-shaped Python interface over the C ABI (include/latsum_b200.h).

Names, argument meaning and error behaviour follow the reference's C++ API
(/root/reference/proj/include/latsum):

=====================================  =========================================
this module                            reference
=====================================  =========================================
`build_reference_canonical`            reference.hpp:95-153
`assembled_sum_canonical`              lattice_sum.hpp:198-223
`defected_sum`                         lattice_sum.hpp:339-384 (canonical branch)
`sublattice_union_sum`                 lattice_sum.hpp:411-465
`lattice_sum`                          the above for a generalised `Geometry`
`rhosvd`                               rank_reduction.hpp:176-218
`CanonicalTensor.entry/.to_dense`      canonical.hpp:63-70, :192-202
`TuckerTensor.entry/.to_dense`         tucker.hpp:38-54, :172-178
`TruncationSpec`, `SpectralReport`     rank_reduction.hpp:21-67
=====================================  =========================================

Every tensor lives in device memory behind an opaque handle; host copies are
made only when a method asks for them (``factor``, ``core``, ``to_dense``).
"""
from __future__ import annotations

import ctypes
import os
import weakref
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .workload import NEWTON, YUKAWA, Geometry, from_lattice

__all__ = [
    "Context", "KernelSpec", "TruncationSpec", "SpectralReport", "ReferenceTensor",
    "CanonicalTensor", "TuckerTensor", "build_quadrature", "default_step_constant",
    "reference_shell", "build_reference_canonical", "lattice_sum", "assembled_sum_canonical",
    "defected_sum", "sublattice_union_sum", "rhosvd", "WindowOverflowError", "Geometry",
    "format_spectral_report", "write_spectral_report", "format_provenance", "write_provenance",
]

WindowOverflowError = _lib.WindowOverflowError

DEFLATE = {"never": 0, "always": 1, "auto": 2}


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One CUDA device, stream and cuSOLVER handle (latsum_ctx)."""

    def __init__(self, device: int = 0):
        self._h = ctypes.c_void_p()
        st = _lib.lib().latsum_ctx_create(device, ctypes.byref(self._h))
        if st != 0:
            raise RuntimeError(f"latsum_ctx_create({device}) failed with status {st}: "
                               "a CUDA device is required (no CPU fallback)")
        self.device = device
        # device objects made on this context: close() destroys them first, because their
        # buffers are freed stream-ordered on the context's streams
        self._children = weakref.WeakSet()

    @property
    def handle(self):
        return self._h

    def check(self, st: int):
        _lib.check(st, self._h)

    def synchronize(self):
        self.check(_lib.lib().latsum_ctx_synchronize(self._h))

    def set_host_sink(self, core_ptr: int, core_cap: int, factor_ptrs=(0, 0, 0),
                      factor_caps=(0, 0, 0)):
        """latsum_ctx_set_host_sink: stream the next Tucker results (core chunk by chunk behind
        its contraction, factors first) into host buffers given as raw pointers (pinned
        memory for the overlap) with capacities in doubles; core_ptr = 0 clears the sink."""
        fp = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(int(x)) for x in factor_ptrs])
        fc = _i64(factor_caps)
        self.check(_lib.lib().latsum_ctx_set_host_sink(
            self._h, ctypes.c_void_p(int(core_ptr)) if core_ptr else None, int(core_cap), fp, _p(fc)))

    def set_accumulation(self, order: str = "sliding"):
        """SumOptions.accumulation (lattice_sum.hpp:28-39): "sliding" (default), "ascending" or
        "compensated" for the assemblies made on this context (latsum_ctx_set_accumulation)."""
        self.check(_lib.lib().latsum_ctx_set_accumulation(
            self._h, {"sliding": 0, "ascending": 1, "compensated": 2}[order]))

    def trim_pool(self, keep_bytes: int = 0):
        """Release the unused part of the stream-ordered pool (latsum_ctx_trim_pool)."""
        self.check(_lib.lib().latsum_ctx_trim_pool(self._h, int(keep_bytes)))

    def set_stream(self, stream_ptr: int):
        self.check(_lib.lib().latsum_ctx_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    @property
    def eig_fallbacks(self) -> int:
        """In-house eigensolves redone with cuSOLVER (latsum_ctx_eig_fallbacks)."""
        return int(_lib.lib().latsum_ctx_eig_fallbacks(self._h))

    @property
    def kernel_launches(self) -> int:
        return int(_lib.lib().latsum_ctx_kernel_launches(self._h))

    def init_comm(self, uid: bytes, rank: int, nranks: int):
        """Join a row-sharded multi-GPU group (latsum_ctx_init_comm)."""
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
        self.check(_lib.lib().latsum_ctx_init_comm(self._h, buf, int(rank), int(nranks)))

    @property
    def comm_info(self):
        r, n = ctypes.c_int(), ctypes.c_int()
        _lib.lib().latsum_ctx_comm_info(self._h, ctypes.byref(r), ctypes.byref(n))
        return r.value, n.value

    def set_profiling(self, on: bool):
        self.check(_lib.lib().latsum_ctx_set_profiling(self._h, 1 if on else 0))

    def profile(self) -> dict:
        """{tag: (launches, total_ms, algorithmic_work)} from CUDA events (profiling on)."""
        n = _lib.lib().latsum_ctx_profile(self._h, None, 0)
        if n < 0:
            raise RuntimeError(_lib.lib().latsum_last_error(self._h).decode())
        buf = ctypes.create_string_buffer(int(n) + 1)
        _lib.lib().latsum_ctx_profile(self._h, buf, int(n) + 1)
        out = {}
        for line in buf.value.decode().splitlines():
            tag, cnt, ms, work = line.split()
            out[tag] = (int(cnt), float(ms), float(work))
        return out

    def close(self):
        if self._h:
            for obj in list(getattr(self, "_children", ())):
                obj._destroy()
            _lib.lib().latsum_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _lib.check(_lib.lib().latsum_comm_unique_id(buf))
    return bytes(buf)


def init_comm_from_torch(ctx: Context):
    """One process per GPU under torch.distributed: rank 0's NCCL id is broadcast with
    torch's process group, then every rank joins the library's communicator."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.init_comm(obj[0], rank, world)


class ThreadCollective:
    """Host collectives for ranks that are threads of one process (several contexts, e.g.
    on one device): per channel, every rank deposits its buffer, all wait, and each sums
    (or concatenates) the deposits in rank order, so every rank gets bit-identical results."""

    def __init__(self, nranks: int):
        import threading
        self.n = nranks
        self._lock = threading.Lock()
        self._slots = {}  # channel -> (barrier, deposits)

    def _slot(self, channel):
        import threading
        with self._lock:
            if channel not in self._slots:
                self._slots[channel] = (threading.Barrier(self.n), [None] * self.n)
            return self._slots[channel]

    def allreduce(self, rank: int, channel: int, buf: np.ndarray):
        bar, dep = self._slot(channel)
        dep[rank] = buf.copy()
        bar.wait()
        if os.environ.get("LATSUM_COLL_DEBUG"):
            print(f"[coll] rank {rank} ch {channel} n {buf.size} sums "
                  f"{[float(np.sum(d)) for d in dep]}", flush=True)
        acc = dep[0].copy()
        for q in range(1, self.n):
            acc += dep[q]
        bar.wait()
        buf[:] = acc

    def allgather(self, rank: int, channel: int, send: np.ndarray, recv: np.ndarray):
        bar, dep = self._slot(channel)
        dep[rank] = send.copy()
        bar.wait()
        recv[:] = np.concatenate(dep)
        bar.wait()


class TorchCollective:
    """Host collectives over torch.distributed (gloo): one process group per channel so the
    library's concurrent worker streams never interleave on one group."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.groups = [dist.new_group(backend="gloo") for _ in range(5)]

    def allreduce(self, rank: int, channel: int, buf: np.ndarray):
        import torch
        t = torch.from_numpy(buf)
        self.dist.all_reduce(t, group=self.groups[channel])

    def allgather(self, rank: int, channel: int, send: np.ndarray, recv: np.ndarray):
        import torch
        n = send.size
        outs = [torch.empty(n, dtype=torch.float64) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(outs, torch.from_numpy(send.copy()), group=self.groups[channel])
        recv[:] = torch.cat(outs).numpy()


def init_host_comm(ctx: Context, rank: int, nranks: int, collective) -> None:
    """latsum_ctx_init_host_comm: run the row-sharded reduction (the NCCL path's partial
    products, all-reduces and all-gathers) over `collective` (ThreadCollective,
    TorchCollective or anything with the same allreduce / allgather methods)."""

    def ar(user, channel, ptr, count):
        try:
            collective.allreduce(rank, channel, np.ctypeslib.as_array(ptr, shape=(count,)))
            return 0
        except Exception:  # reported to the library as a failed collective
            return 1

    def ag(user, channel, sptr, rptr, count):
        try:
            collective.allgather(rank, channel, np.ctypeslib.as_array(sptr, shape=(count,)),
                                 np.ctypeslib.as_array(rptr, shape=(count * nranks,)))
            return 0
        except Exception:
            return 1

    cb = (_lib.HOST_ALLREDUCE(ar), _lib.HOST_ALLGATHER(ag))
    ctx._host_comm = cb  # the callbacks live as long as the context
    ctx.check(_lib.lib().latsum_ctx_init_host_comm(ctx.handle, int(rank), int(nranks),
                                                   ctypes.cast(cb[0], ctypes.c_void_p),
                                                   ctypes.cast(cb[1], ctypes.c_void_p), None))


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ----------------------------------------------------------------------------- specs

@dataclass(frozen=True)
class KernelSpec:
    """kernel.hpp:37-152 restricted to the hot path's gauss-type primitives."""
    family: int = NEWTON
    lam: float = 0.0

    @staticmethod
    def newton() -> "KernelSpec":
        return KernelSpec(NEWTON, 0.0)

    @staticmethod
    def yukawa(lam: float) -> "KernelSpec":
        if not lam > 0.0:
            raise ValueError("yukawa lambda must be positive")
        return KernelSpec(YUKAWA, float(lam))


@dataclass
class TruncationSpec:
    """rank_reduction.hpp:21-43."""
    ranks: Optional[Tuple[int, int, int]] = None
    tolerance: Optional[float] = None

    def validate(self):
        if self.ranks is None and self.tolerance is None:
            raise ValueError("TruncationSpec: need ranks or tolerance")
        if self.tolerance is not None and not (0.0 < self.tolerance < 1.0):
            raise ValueError("TruncationSpec: tolerance must lie in (0,1)")

    @staticmethod
    def fixed_ranks(r1: int, r2: int, r3: int) -> "TruncationSpec":
        return TruncationSpec(ranks=(int(r1), int(r2), int(r3)))

    @staticmethod
    def tol(eps: float) -> "TruncationSpec":
        return TruncationSpec(tolerance=float(eps))


@dataclass
class SpectralReport:
    """rank_reduction.hpp:49-67 plus the GPU path's diagnostics and stage timings."""
    singular_values: list
    chosen_ranks: Tuple[int, int, int]
    bound_abs: float
    bound_rel: float
    weight_norm: float
    input_norm: float
    stability_constant: float
    stability_ok: bool
    tie_at_cutoff: Tuple[bool, bool, bool]
    cutoff_margin: Tuple[float, float, float]
    deflated: Tuple[bool, bool, bool]
    gram_rows: Tuple[bool, bool, bool]
    gram_size: Tuple[int, int, int]
    ms: dict
    deflate_k1: Tuple[int, int, int] = (0, 0, 0)

    def tail(self, mode: int) -> float:
        sv = self.singular_values[mode]
        return float(np.sqrt(np.sum(sv[self.chosen_ranks[mode]:] ** 2)))


# ----------------------------------------------------------------------------- host rules

def build_quadrature(kernel: KernelSpec, M: int, step_constant: float, shell) -> Tuple[np.ndarray, np.ndarray]:
    R = 2 * M + 1
    t, a = np.zeros(R), np.zeros(R)
    _lib.check(_lib.lib().latsum_build_quadrature(kernel.family, kernel.lam, M, step_constant,
                                                  shell[0], shell[1], _p(t), _p(a)))
    return t, a


def default_step_constant(kernel: KernelSpec, M: int, shell, npts: int = 320) -> float:
    return float(_lib.lib().latsum_default_step_constant(kernel.family, kernel.lam, M, shell[0],
                                                         shell[1], npts))


def reference_shell(N, box) -> Tuple[float, float]:
    out = np.zeros(2)
    _lib.lib().latsum_reference_shell(_p(_i64(N)), _p(_f64(box)), _p(out))
    return float(out[0]), float(out[1])


# ----------------------------------------------------------------------------- tensors

class ReferenceTensor:
    """reference.hpp:65-80 (doubled grid, canonical form, device resident)."""

    def __init__(self, ctx: Context, handle, kernel: KernelSpec, N, box, M):
        self.ctx, self._h, self.kernel = ctx, handle, kernel
        ctx._children.add(self)
        self.N, self.box, self.M = tuple(int(n) for n in N), tuple(float(b) for b in box), M
        rank, c0, shell = ctypes.c_int(), ctypes.c_double(), np.zeros(2)
        _lib.lib().latsum_reference_info(self._h, ctypes.byref(rank), ctypes.byref(c0), _p(shell))
        self.rank, self.step_constant, self.shell = rank.value, c0.value, (shell[0], shell[1])

    @property
    def handle(self):
        return self._h

    def factor(self, mode: int) -> np.ndarray:
        out = np.zeros((2 * self.N[mode], self.rank), order="F")
        self.ctx.check(_lib.lib().latsum_reference_factor(self.ctx.handle, self._h, mode, _p(out)))
        return out

    @property
    def weights(self) -> np.ndarray:
        w = np.zeros(self.rank)
        _lib.check(_lib.lib().latsum_reference_weights(self._h, _p(w)))
        return w

    def quadrature(self):
        t, a = np.zeros(self.rank), np.zeros(self.rank)
        _lib.check(_lib.lib().latsum_reference_quadrature(self._h, _p(t), _p(a)))
        return t, a

    def _destroy(self):
        if getattr(self, "_h", None):
            _lib.lib().latsum_reference_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self._destroy()
        except Exception:  # interpreter shutdown
            pass


def build_reference_canonical(kernel: KernelSpec, N: Sequence[int], box: Sequence[float], M: int,
                              step_constant: float = 0.0,
                              ctx: Optional[Context] = None) -> ReferenceTensor:
    """reference.hpp:95-153 with the grid given as (cells N_l, box widths b_l)."""
    ctx = ctx or default_context()
    h = ctypes.c_void_p()
    ctx.check(_lib.lib().latsum_reference_build(ctx.handle, kernel.family, kernel.lam,
                                                _p(_i64(N)), _p(_f64(box)), int(M),
                                                float(step_constant), ctypes.byref(h)))
    return ReferenceTensor(ctx, h, kernel, N, box, M)


class CanonicalTensor:
    """canonical.hpp:19-202: unit side-matrix columns + weights, device resident.

    Internally the side matrices are stored as per-mode dictionaries of distinct
    columns; `factor(mode)` materialises the reference's N x M_c form."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self._h = ctx, handle
        ctx._children.add(self)
        dims, dcols, rank = np.zeros(3, np.int64), np.zeros(3, np.int64), ctypes.c_int64()
        # merged_terms is not requested here: it waits for the host-side term merge that
        # the library overlaps with the RHOSVD's first kernels
        _lib.lib().latsum_canonical_info(self._h, _p(dims), ctypes.byref(rank), _p(dcols), None)
        self.dims = tuple(int(x) for x in dims)
        self.rank = int(rank.value)
        self.dict_cols = tuple(int(x) for x in dcols)

    @property
    def merged_terms(self) -> int:
        """Rank-1 terms left after merging identical ones (t and -t, repeated sites)."""
        T = ctypes.c_int64()
        st = _lib.lib().latsum_canonical_info(self._h, None, None, None, ctypes.byref(T))
        _lib.check(st)  # a failed background term merge surfaces here, not as 0 terms
        return int(T.value)

    @property
    def handle(self):
        return self._h

    @property
    def weights(self) -> np.ndarray:
        w = np.zeros(self.rank)
        _lib.check(_lib.lib().latsum_canonical_weights(self._h, _p(w)))
        return w

    def factor(self, mode: int) -> np.ndarray:
        out = np.zeros((self.dims[mode], self.rank), order="F")
        self.ctx.check(_lib.lib().latsum_canonical_factor(self.ctx.handle, self._h, mode, _p(out)))
        return out

    def factor_device(self, mode: int, out_ptr: int):
        self.ctx.check(_lib.lib().latsum_canonical_factor_device(self.ctx.handle, self._h, mode,
                                                                 ctypes.c_void_p(out_ptr)))

    def entries(self, probes) -> np.ndarray:
        pr = _i64(probes).reshape(-1, 3)
        out = np.zeros(pr.shape[0])
        self.ctx.check(_lib.lib().latsum_canonical_entries(self.ctx.handle, self._h, _p(pr),
                                                           pr.shape[0], _p(out)))
        return out

    def entry(self, i: int, j: int, k: int) -> float:
        return float(self.entries([[i, j, k]])[0])

    def norm(self) -> float:
        v = ctypes.c_double()
        self.ctx.check(_lib.lib().latsum_canonical_norm(self.ctx.handle, self._h, ctypes.byref(v)))
        return v.value

    def eval_box_device(self, lo, hi, out_ptr: int):
        self.ctx.check(_lib.lib().latsum_canonical_eval_box_device(
            self.ctx.handle, self._h, _p(_i64(lo)), _p(_i64(hi)), ctypes.c_void_p(out_ptr)))

    def to_dense(self, lo=None, hi=None, guard: int = 10_000_000) -> np.ndarray:
        """canonical.hpp:192-202 on a box (default: the whole grid), via the device."""
        import torch
        lo = (0, 0, 0) if lo is None else tuple(lo)
        hi = self.dims if hi is None else tuple(hi)
        shape = tuple(h - l for l, h in zip(lo, hi))
        if int(np.prod(shape)) > guard:
            raise OverflowError(f"dense materialization of {int(np.prod(shape))} entries exceeds "
                                f"the guard limit {guard}")
        buf = torch.empty(int(np.prod(shape)), dtype=torch.float64, device=f"cuda:{self.ctx.device}")
        self.eval_box_device(lo, hi, buf.data_ptr())
        self.ctx.synchronize()
        return buf.cpu().numpy().reshape(shape, order="F")

    def _destroy(self):
        if getattr(self, "_h", None):
            _lib.lib().latsum_canonical_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self._destroy()
        except Exception:  # interpreter shutdown
            pass


class TuckerTensor:
    """tucker.hpp:19-73, device resident."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self._h = ctx, handle
        ctx._children.add(self)
        dims, ranks = np.zeros(3, np.int64), np.zeros(3, np.int64)
        _lib.lib().latsum_tucker_info(self._h, _p(dims), _p(ranks))
        self.dims = tuple(int(x) for x in dims)
        self.ranks = tuple(int(x) for x in ranks)

    @property
    def handle(self):
        return self._h

    @property
    def sink_written(self) -> bool:
        """The core and factors were streamed to the context's host sink."""
        return bool(_lib.lib().latsum_tucker_sink_written(self._h))

    @property
    def has_core(self) -> bool:
        return bool(_lib.lib().latsum_tucker_has_core(self._h))

    def core_slab(self):
        """(a0, slab): this rank's rows [a0, a0 + ra) of mode 1 of the core (rhosvd(...,
        core_slabs=True) on a sharded context; the whole core otherwise)."""
        a0, ra = ctypes.c_int64(), ctypes.c_int64()
        L = _lib.lib()
        self.ctx.check(L.latsum_tucker_core_slab(self.ctx.handle, self._h, ctypes.byref(a0),
                                                 ctypes.byref(ra), None))
        out = np.zeros((ra.value, self.ranks[1], self.ranks[2]), order="F")
        self.ctx.check(L.latsum_tucker_core_slab(self.ctx.handle, self._h, ctypes.byref(a0),
                                                 ctypes.byref(ra), _p(out)))
        return int(a0.value), out

    @property
    def core(self) -> np.ndarray:
        out = np.zeros(self.ranks, order="F")
        self.ctx.check(_lib.lib().latsum_tucker_core(self.ctx.handle, self._h, _p(out)))
        return out

    def factor(self, mode: int) -> np.ndarray:
        out = np.zeros((self.dims[mode], self.ranks[mode]), order="F")
        self.ctx.check(_lib.lib().latsum_tucker_factor(self.ctx.handle, self._h, mode, _p(out)))
        return out

    def projected_form(self):
        """Factors-only tensors (no dense core): (P_l (r_l x d_l) per mode, term columns
        (T x 3, int32), term weights (T)) with V = sum_t w_t prod_l (U_l P_l)[i_l, c_l(t)]."""
        d, T = np.zeros(3, np.int64), ctypes.c_int64()
        L = _lib.lib()
        self.ctx.check(L.latsum_tucker_projected_form(self.ctx.handle, self._h, _p(d),
                                                      ctypes.byref(T), *([None] * 7)))
        P = [np.zeros((self.ranks[l], int(d[l])), order="F") for l in range(3)]
        tc = [np.zeros(T.value, np.int32) for _ in range(3)]
        w = np.zeros(T.value)
        self.ctx.check(L.latsum_tucker_projected_form(
            self.ctx.handle, self._h, _p(d), ctypes.byref(T), _p(P[0]), _p(P[1]), _p(P[2]),
            _p(tc[0]), _p(tc[1]), _p(tc[2]), _p(w)))
        return P, np.stack(tc, axis=1), w

    def entries(self, probes) -> np.ndarray:
        pr = _i64(probes).reshape(-1, 3)
        out = np.zeros(pr.shape[0])
        self.ctx.check(_lib.lib().latsum_tucker_entries(self.ctx.handle, self._h, _p(pr),
                                                        pr.shape[0], _p(out)))
        return out

    def entry(self, i: int, j: int, k: int) -> float:
        return float(self.entries([[i, j, k]])[0])

    def eval_box_device(self, lo, hi, out_ptr: int):
        self.ctx.check(_lib.lib().latsum_tucker_eval_box_device(
            self.ctx.handle, self._h, _p(_i64(lo)), _p(_i64(hi)), ctypes.c_void_p(out_ptr)))

    def to_dense(self, lo=None, hi=None, guard: int = 10_000_000) -> np.ndarray:
        """tucker.hpp:172-178 on a box (default: the whole grid) into host memory."""
        lo = (0, 0, 0) if lo is None else tuple(lo)
        hi = self.dims if hi is None else tuple(hi)
        shape = tuple(h - l for l, h in zip(lo, hi))
        if int(np.prod(shape)) > guard:
            raise OverflowError(f"dense materialization of {int(np.prod(shape))} entries exceeds "
                                f"the guard limit {guard}")
        out = np.zeros(shape, order="F")
        self.ctx.check(_lib.lib().latsum_tucker_eval_box(self.ctx.handle, self._h, _p(_i64(lo)),
                                                         _p(_i64(hi)), _p(out)))
        return out

    def _destroy(self):
        if getattr(self, "_h", None):
            _lib.lib().latsum_tucker_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self._destroy()
        except Exception:  # interpreter shutdown
            pass


# ----------------------------------------------------------------------------- sums

def _shift_tables(geom: Geometry):
    nsub = len(geom.sublattices)
    counts = np.array([[len(s.shifts[l]) for l in range(3)] for s in geom.sublattices],
                      np.int64).reshape(-1, 3)
    shifts = (np.concatenate([np.asarray(s.shifts[l], np.int64) for s in geom.sublattices
                              for l in range(3)]) if nsub else np.zeros(0, np.int64))
    charges = np.array([s.charge for s in geom.sublattices], np.float64)
    return nsub, _i64(counts), _i64(shifts), _f64(charges), _i64(geom.defect_shifts.reshape(-1, 3)), \
        _f64(geom.defect_charges)


def _block_tables(geom: Geometry):
    """Ordered product blocks (latsum_canonical_assemble_blocks): counts nblk x 3, the
    shift lists concatenated in (block, mode) order, one charge per block."""
    if geom.defect_blocks is None:  # sublattices, then single sites (vectorised: cfg5 has 1000)
        subs = geom.sublattices
        nd = geom.defect_shifts.shape[0]
        counts = np.ones((len(subs) + nd, 3), np.int64)
        for i, b in enumerate(subs):
            counts[i] = [len(b.shifts[l]) for l in range(3)]
        parts = [np.asarray(b.shifts[l], np.int64) for b in subs for l in range(3)]
        parts.append(np.asarray(geom.defect_shifts, np.int64).reshape(-1))
        charges = np.concatenate([np.array([b.charge for b in subs], np.float64),
                                  np.asarray(geom.defect_charges, np.float64)])
        return len(subs) + nd, _i64(counts), _i64(np.concatenate(parts)), _f64(charges)
    blocks = geom.blocks()
    counts = np.array([[len(b.shifts[l]) for l in range(3)] for b in blocks],
                      np.int64).reshape(-1, 3)
    shifts = (np.concatenate([np.asarray(b.shifts[l], np.int64) for b in blocks
                              for l in range(3)]) if blocks else np.zeros(0, np.int64))
    charges = np.array([b.charge for b in blocks], np.float64)
    return len(blocks), _i64(counts), _i64(shifts), _f64(charges)


def lattice_sum(ref: ReferenceTensor, geom: Geometry) -> CanonicalTensor:
    """Assembled sublattice sums plus additive defect blocks (canonical, untruncated):
    lattice_sum.hpp:198-223, :339-384 canonical branch without a spec; product-structure
    defect clusters stay at reference rank (:316-321)."""
    ctx = ref.ctx
    nblk, counts, shifts, charges = _block_tables(geom)
    h = ctypes.c_void_p()
    ctx.check(_lib.lib().latsum_canonical_assemble_blocks(
        ctx.handle, ref.handle, nblk, _p(counts), _p(shifts), _p(charges), ctypes.byref(h)))
    return CanonicalTensor(ctx, h)


def assembled_sum_canonical(ref: ReferenceTensor, cells, n_per_cell: int, cell_width: float = 1.0,
                            base_charge: float = 1.0, active=None) -> CanonicalTensor:
    """lattice_sum.hpp:198-223 for LatticeGeometry(cells, cell_width) on lattice_grid."""
    g = from_lattice(cells, n_per_cell, cell_width, base_charge=base_charge, active=active,
                     M=ref.M)
    return lattice_sum(ref, g)


def defected_sum(ref: ReferenceTensor, cells, n_per_cell: int, defects, cell_width: float = 1.0,
                 base_charge: float = 1.0, spec: Optional[TruncationSpec] = None, deflate="auto",
                 refs: Optional[Sequence[ReferenceTensor]] = None):
    """lattice_sum.hpp:339-400 (canonical branch): base lattice + defect clusters
    `defects` = [(sites, charge, grid_offset)], truncated by RHOSVD when `spec` is set.

    A defect given as (sites, charge, grid_offset, KernelSpec) carries its own kernel
    (DefectSpec.kernel, lattice_sum.hpp:301-303); `refs` (the ReferenceSet, :260-276) must then
    hold that kernel's reference tensor on the same grid.  Every maximal run of clusters sharing
    a kernel is assembled against its reference and added with `add_concat` in DefectSpec order,
    the terms the reference's per-cluster add_concat loop (:372-374) produces."""
    base_k = ref.kernel

    def kernel_of(d):
        return d[3] if len(d) > 3 and d[3] is not None else base_k

    def find(k):
        for r in [ref] + list(refs or ()):
            if r.kernel == k:
                return r
        raise ValueError(f"defected_sum: no reference tensor for kernel {k}")

    for d in defects:
        if not len(d[0]):
            raise ValueError("defected_sum: defect with no sites")
        find(kernel_of(d))
    runs = []
    for d in defects:
        k = kernel_of(d)
        if runs and runs[-1][0] == k:
            runs[-1][1].append(tuple(d[:3]))
        else:
            runs.append((k, [tuple(d[:3])]))
    lead = runs.pop(0)[1] if runs and runs[0][0] == base_k else []
    g = from_lattice(cells, n_per_cell, cell_width, base_charge=base_charge, defects=lead, M=ref.M)
    can = lattice_sum(ref, g)
    for k, ds in runs:
        rk = find(k)
        gk = from_lattice(cells, n_per_cell, cell_width, family=k.family, lam=k.lam,
                          base_charge=base_charge, defects=ds, sublattices=[], parent_cells=cells,
                          M=rk.M)
        can = add_concat(can, lattice_sum(rk, gk))
    if spec is None:
        return can
    return rhosvd(can, spec, deflate=deflate)


def sublattice_union_sum(ref: ReferenceTensor, parent_cells, n_per_cell: int, subs,
                         cell_width: float = 1.0, spec: Optional[TruncationSpec] = None,
                         deflate="auto"):
    """lattice_sum.hpp:411-465; subs = [(cells, offset_cells)]."""
    g = from_lattice(parent_cells, n_per_cell, cell_width, sublattices=subs,
                     parent_cells=parent_cells, M=ref.M)
    can = lattice_sum(ref, g)
    if spec is None:
        return can
    return rhosvd(can, spec, deflate=deflate)


def rhosvd(can: CanonicalTensor, spec: TruncationSpec, deflate: str = "auto",
           form_core: bool = True, core_slabs: bool = False):
    """rank_reduction.hpp:176-218 -> (TuckerTensor, SpectralReport).

    form_core=False keeps the projected factors instead of the dense r1 x r2 x r3 core
    (LATSUM_RHOSVD_FACTORS_ONLY); entries / boxes are then evaluated in projected-CP
    form, equal to the Tucker tensor (BASELINE cfg5: the core would be 518 GB)."""
    spec.validate()
    ctx = can.ctx
    rep = _lib.LatsumReport()
    h = ctypes.c_void_p()
    ranks = _i64(spec.ranks) if spec.ranks is not None else None
    ctx.check(_lib.lib().latsum_rhosvd_ex(ctx.handle, can.handle,
                                          _p(ranks) if ranks is not None else None,
                                          float(spec.tolerance or 0.0), DEFLATE[deflate],
                                          (0 if form_core else 1) | (2 if core_slabs else 0),
                                          ctypes.byref(h),
                                          ctypes.byref(rep)))
    t = TuckerTensor(ctx, h)
    sv = []
    for l in range(3):
        s = np.zeros(int(rep.n_singular[l]))
        _lib.check(_lib.lib().latsum_tucker_singular_values(h, l, _p(s)))
        sv.append(s)
    report = SpectralReport(
        singular_values=sv, chosen_ranks=tuple(int(x) for x in rep.chosen_ranks),
        bound_abs=rep.bound_abs, bound_rel=rep.bound_rel, weight_norm=rep.weight_norm,
        input_norm=rep.input_norm, stability_constant=rep.stability_constant,
        stability_ok=bool(rep.stability_ok), tie_at_cutoff=tuple(bool(x) for x in rep.tie_at_cutoff),
        cutoff_margin=tuple(float(x) for x in rep.cutoff_margin),
        deflated=tuple(bool(x) for x in rep.deflated), gram_rows=tuple(bool(x) for x in rep.gram_rows),
        gram_size=tuple(int(x) for x in rep.gram_size),
        ms=dict(gram=rep.ms_gram, syevd=rep.ms_syevd, deflate=rep.ms_deflate,
                project=rep.ms_project, core=rep.ms_core, norm=rep.ms_norm, total=rep.ms_total),
        deflate_k1=tuple(int(x) for x in rep.deflate_k1))
    return t, report


def oracle_entries(ref: ReferenceTensor, geom: Geometry, probes) -> np.ndarray:
    """lattice_sum.hpp:656-671 brute-force windowed sum over every source of `geom`
    (enumerate_sources order) at the probes, computed on the device."""
    shifts, w = geom.sources()
    pr = _i64(probes).reshape(-1, 3)
    out = np.zeros(pr.shape[0])
    ref.ctx.check(_lib.lib().latsum_verify_entries(ref.ctx.handle, ref.handle, shifts.shape[0],
                                                   _p(shifts), _p(_f64(w)), _p(pr), pr.shape[0],
                                                   _p(out)))
    return out


def verify_probes(seed: int, dims, count: int) -> np.ndarray:
    """commands.cpp:254-260: the probe points `latsum verify` draws for `seed`
    (std::mt19937_64 + uniform_int_distribution per mode; latsum_verify_probes)."""
    d = _i64(dims)
    out = np.zeros((int(count), 3), np.int64)
    _lib.lib().latsum_verify_probes(ctypes.c_uint64(int(seed) & (2 ** 64 - 1)), _p(d), int(count), _p(out))
    return out


def verify(tensor, ref: ReferenceTensor, geom: Geometry, probes=500, seed: int = 0,
           tolerance: Optional[float] = None, bound_abs: Optional[float] = None) -> dict:
    """cmd_verify (commands.cpp:200-284): max|got - oracle| / max|oracle| over seeded
    probes, gated by the recorded truncation bound if given, else by `tolerance`."""
    if np.isscalar(probes):
        probes = verify_probes(seed, geom.N, int(probes))
    pr = _i64(probes).reshape(-1, 3)
    want = oracle_entries(ref, geom, pr)
    got = tensor.entries(pr)
    max_abs = float(np.max(np.abs(got - want)))
    max_mag = float(np.max(np.abs(want)))
    rel = max_abs / max_mag if max_mag > 0 else max_abs
    ok = (max_abs <= bound_abs) if bound_abs is not None else (
        rel <= tolerance if tolerance is not None else True)
    return dict(probes=int(pr.shape[0]), max_abs=max_abs, max_oracle=max_mag, normalized=rel,
                ok=bool(ok))


def canonical_to_tucker(can: CanonicalTensor, spec: TruncationSpec, max_als_sweeps: int = 30,
                        als_stagnation_tol: float = 1e-8):
    """rank_reduction.hpp:280-306: rhosvd + ALS refinement + shrink_core (tolerance mode)
    -> (TuckerTensor, SpectralReport, als_sweeps)."""
    spec.validate()
    ctx = can.ctx
    rep = _lib.LatsumReport()
    h = ctypes.c_void_p()
    sweeps = ctypes.c_int()
    ranks = _i64(spec.ranks) if spec.ranks is not None else None
    ctx.check(_lib.lib().latsum_canonical_to_tucker(
        ctx.handle, can.handle, _p(ranks) if ranks is not None else None,
        float(spec.tolerance or 0.0), int(max_als_sweeps), float(als_stagnation_tol),
        ctypes.byref(h), ctypes.byref(rep), ctypes.byref(sweeps)))
    t = TuckerTensor(ctx, h)
    sv = []
    for l in range(3):
        s = np.zeros(int(rep.n_singular[l]))
        _lib.check(_lib.lib().latsum_tucker_singular_values(h, l, _p(s)))
        sv.append(s)
    report = SpectralReport(
        singular_values=sv, chosen_ranks=tuple(int(x) for x in rep.chosen_ranks),
        bound_abs=rep.bound_abs, bound_rel=rep.bound_rel, weight_norm=rep.weight_norm,
        input_norm=rep.input_norm, stability_constant=rep.stability_constant,
        stability_ok=bool(rep.stability_ok), tie_at_cutoff=tuple(bool(x) for x in rep.tie_at_cutoff),
        cutoff_margin=tuple(float(x) for x in rep.cutoff_margin),
        deflated=tuple(bool(x) for x in rep.deflated), gram_rows=tuple(bool(x) for x in rep.gram_rows),
        gram_size=tuple(int(x) for x in rep.gram_size), ms={})
    return t, report, int(sweeps.value)


def canonical_from_arrays(weights, factors, ctx: Optional[Context] = None) -> CanonicalTensor:
    """CanonicalTensor(dims, weights, factors) (canonical.hpp:25-29): unit columns as given."""
    ctx = ctx or default_context()
    w = _f64(weights)
    F = [np.asfortranarray(f, dtype=np.float64) for f in factors]
    dims = _i64([f.shape[0] for f in F])
    h = ctypes.c_void_p()
    ctx.check(_lib.lib().latsum_canonical_from_host(ctx.handle, _p(dims), w.size, _p(w), _p(F[0]),
                                                    _p(F[1]), _p(F[2]), ctypes.byref(h)))
    return CanonicalTensor(ctx, h)


def add_concat(a: CanonicalTensor, b: CanonicalTensor) -> CanonicalTensor:
    """canonical.hpp:94-110: a + b by concatenation (a's terms first).  A defect cluster with its
    own kernel (lattice_sum.hpp:301-303) is `lattice_sum(reference of that kernel, geometry of the
    cluster alone)` added with this, in DefectSpec order, as defected_sum does (:372-374)."""
    h = ctypes.c_void_p()
    a.ctx.check(_lib.lib().latsum_canonical_concat(a.ctx.handle, a.handle, b.handle, ctypes.byref(h)))
    return CanonicalTensor(a.ctx, h)


def write_tensor(path: str, tensor):
    """tensor_io.cpp:45-76 ("LTSTNSR" v1 + FNV-1a-64), from device-resident tensors."""
    ctx = tensor.ctx
    can = tensor.handle if isinstance(tensor, CanonicalTensor) else None
    tk = tensor.handle if isinstance(tensor, TuckerTensor) else None
    ctx.check(_lib.lib().latsum_tensor_write(ctx.handle, can, tk, str(path).encode()))


def read_tensor(path: str, ctx: Optional[Context] = None):
    """tensor_io.cpp:78-129: checksum-guarded read into a device-resident tensor."""
    ctx = ctx or default_context()
    hc, ht = ctypes.c_void_p(), ctypes.c_void_p()
    ctx.check(_lib.lib().latsum_tensor_read(ctx.handle, str(path).encode(), ctypes.byref(hc),
                                            ctypes.byref(ht)))
    return CanonicalTensor(ctx, hc) if hc.value else TuckerTensor(ctx, ht)


def reference_for(geom: Geometry, ctx: Optional[Context] = None) -> ReferenceTensor:
    kernel = KernelSpec(geom.family, geom.lam)
    return build_reference_canonical(kernel, geom.N, geom.box, geom.M, geom.C0, ctx=ctx)


def sum_to_tucker(geom: Geometry, tolerance: float, ctx: Optional[Context] = None):
    """cmd_sum's defected/sublattice path with a tolerance (commands.cpp:108-179) in one
    C-ABI call with host-resident inputs: stages 1-3, Tucker result on the device."""
    ctx = ctx or default_context()
    if geom.defect_blocks is None:
        nsub, counts, shifts, charges, dsh, dch = _shift_tables(geom)
    else:  # ordered product blocks, all passed as sublattice-style blocks (same layout)
        nsub, counts, shifts, charges = _block_tables(geom)
        dsh, dch = _i64(np.zeros((0, 3), np.int64)), _f64(np.zeros(0))
    rep = _lib.LatsumReport()
    h = ctypes.c_void_p()
    ctx.check(_lib.lib().latsum_sum_to_tucker(
        ctx.handle, geom.family, geom.lam, _p(_i64(geom.N)), _p(_f64(geom.box)), geom.M, geom.C0,
        nsub, _p(counts), _p(shifts), _p(charges), dsh.shape[0], _p(dsh), _p(dch),
        float(tolerance), ctypes.byref(h), ctypes.byref(rep)))
    return TuckerTensor(ctx, h), rep


# ----------------------------------------------------------------------------- reports

def _format(fn, *args) -> str:
    n = fn(*args, None, 0)
    if n < 0:
        raise ValueError("report formatting: null argument")
    buf = ctypes.create_string_buffer(int(n) + 1)
    fn(*args, buf, int(n) + 1)
    return buf.raw[:n].decode()


def format_spectral_report(report: SpectralReport) -> str:
    """report.cpp:28-46 write_spectral_report (latsum_format_spectral_report)."""
    r = _lib.LatsumReport()
    sv = [np.ascontiguousarray(np.asarray(report.singular_values[l], np.float64)) for l in range(3)]
    for l in range(3):
        r.chosen_ranks[l] = int(report.chosen_ranks[l])
        r.tie_at_cutoff[l] = int(bool(report.tie_at_cutoff[l]))
        r.n_singular[l] = sv[l].size
    r.bound_abs, r.bound_rel = float(report.bound_abs), float(report.bound_rel)
    r.weight_norm, r.input_norm = float(report.weight_norm), float(report.input_norm)
    r.stability_constant = float(report.stability_constant)
    r.stability_ok = int(bool(report.stability_ok))
    ptrs = (ctypes.c_void_p * 3)(*[x.ctypes.data for x in sv])
    return _format(_lib.lib().latsum_format_spectral_report, ctypes.byref(r), ptrs)


def write_spectral_report(path: str, report: SpectralReport) -> None:
    """commands.cpp:67-71: the report file next to the tensor."""
    with open(path, "w") as f:
        f.write(format_spectral_report(report))


def format_provenance(geom: Geometry, tensor, report: Optional[SpectralReport] = None,
                      seed: Optional[int] = None, extra_lines: Sequence[str] = ()) -> str:
    """report.cpp:48-73 write_provenance for the result `tensor` (CanonicalTensor or
    TuckerTensor) of the sum described by `geom` (latsum_format_provenance)."""
    p = _lib.LatsumProvenance()
    p.seed = int(geom.seed if seed is None else seed) & (2 ** 64 - 1)
    cells = geom.cell_counts()
    for l in range(3):
        p.grid[l] = int(geom.N[l])
        p.cells[l] = int(cells[l])
    if isinstance(tensor, TuckerTensor) or (hasattr(tensor, "ranks") and not hasattr(tensor, "rank")):
        p.format = 1
        for l in range(3):
            p.ranks[l] = int(tensor.ranks[l])
    else:
        p.format = 0
        p.rank = int(tensor.rank)
    summ = geom.summands()
    p.nsummands = len(summ)
    labels = (ctypes.c_char_p * max(1, len(summ)))(*[x[0].encode() for x in summ])
    ranks = np.ascontiguousarray([x[1] for x in summ] or [0], np.int64)
    sites = np.ascontiguousarray([x[2] for x in summ] or [0], np.int64)
    p.labels = ctypes.cast(labels, ctypes.POINTER(ctypes.c_char_p))
    p.summand_ranks = ranks.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    p.summand_sites = sites.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    if report is not None:
        p.has_report = 1
        p.bound_abs, p.bound_rel = float(report.bound_abs), float(report.bound_rel)
    extra = (ctypes.c_char_p * max(1, len(extra_lines)))(*[x.encode() for x in extra_lines])
    p.nextra = len(extra_lines)
    p.extra = ctypes.cast(extra, ctypes.POINTER(ctypes.c_char_p))
    return _format(_lib.lib().latsum_format_provenance, ctypes.byref(p))


def write_provenance(path: str, geom: Geometry, tensor, report: Optional[SpectralReport] = None,
                     seed: Optional[int] = None, extra_lines: Sequence[str] = ()) -> None:
    """commands.cpp:62-66: the provenance sidecar."""
    with open(path, "w") as f:
        f.write(format_provenance(geom, tensor, report, seed, extra_lines))

