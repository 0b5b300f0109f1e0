"""ctypes binding of include/latsum_b200.h (liblatsum_b200.so, built in-tree).

There is no CPU fallback: importing the product without the built library, or
calling a compute entry point without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblatsum_b200.so")
CSRC = os.path.join(HERE, "csrc")

OK = 0
ERRORS = {
    1: ValueError,        # std::invalid_argument
    2: IndexError,        # WindowOverflowError (std::out_of_range)
    3: RuntimeError,      # CUDA
    4: RuntimeError,      # cuSOLVER
    5: MemoryError,
    6: OverflowError,     # std::length_error (dense guard)
    7: NotImplementedError,
    8: RuntimeError,      # NCCL
    9: IOError,           # TensorIoError
}


class WindowOverflowError(IndexError):
    """grid.hpp:87-98 WindowOverflowError; `.mode` is 1-based."""

    def __init__(self, msg: str):
        super().__init__(msg)
        self.mode = 0
        for tok in msg.split():
            if tok.rstrip(":").isdigit():
                self.mode = int(tok.rstrip(":"))
                break


class LatsumReport(ctypes.Structure):
    _fields_ = [
        ("chosen_ranks", ctypes.c_int64 * 3),
        ("bound_abs", ctypes.c_double), ("bound_rel", ctypes.c_double),
        ("weight_norm", ctypes.c_double), ("input_norm", ctypes.c_double),
        ("stability_constant", ctypes.c_double),
        ("stability_ok", ctypes.c_int),
        ("tie_at_cutoff", ctypes.c_int * 3),
        ("n_singular", ctypes.c_int64 * 3),
        ("cutoff_margin", ctypes.c_double * 3),
        ("deflated", ctypes.c_int * 3),
        ("gram_rows", ctypes.c_int * 3),
        ("gram_size", ctypes.c_int64 * 3),
        ("ms_gram", ctypes.c_double), ("ms_syevd", ctypes.c_double),
        ("ms_deflate", ctypes.c_double), ("ms_project", ctypes.c_double),
        ("ms_core", ctypes.c_double), ("ms_norm", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("deflate_k1", ctypes.c_int64 * 3),
    ]


# host collectives (latsum_ctx_init_host_comm)
HOST_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_double), ctypes.c_int64)
HOST_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                  ctypes.c_int64)


class LatsumProvenance(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("grid", ctypes.c_int64 * 3), ("cells", ctypes.c_int64 * 3),
        ("format", ctypes.c_int),
        ("rank", ctypes.c_int64), ("ranks", ctypes.c_int64 * 3),
        ("nsummands", ctypes.c_int64),
        ("labels", ctypes.POINTER(ctypes.c_char_p)),
        ("summand_ranks", ctypes.POINTER(ctypes.c_int64)),
        ("summand_sites", ctypes.POINTER(ctypes.c_int64)),
        ("has_report", ctypes.c_int),
        ("bound_abs", ctypes.c_double), ("bound_rel", ctypes.c_double),
        ("nextra", ctypes.c_int64),
        ("extra", ctypes.POINTER(ctypes.c_char_p)),
    ]


# (name, restype, argtypes) for every symbol include/latsum_b200.h declares
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
SIGNATURES = [
    ("latsum_ctx_create", _I, [_I, _P]),
    ("latsum_ctx_destroy", None, [_P]),
    ("latsum_last_error", ctypes.c_char_p, [_P]),
    ("latsum_ctx_set_stream", _I, [_P, _P]),
    ("latsum_ctx_synchronize", _I, [_P]),
    ("latsum_ctx_kernel_launches", _I64, [_P]),
    ("latsum_ctx_eig_fallbacks", _I64, [_P]),
    ("latsum_comm_unique_id", _I, [_P]),
    ("latsum_ctx_init_comm", _I, [_P, _P, _I, _I]),
    ("latsum_ctx_trim_pool", _I, [_P, _I64]),
    ("latsum_ctx_set_host_sink", _I, [_P, _P, _I64, _P, _P]),
    ("latsum_tucker_sink_written", _I, [_P]),
    ("latsum_ctx_init_host_comm", _I, [_P, _I, _I, _P, _P, _P]),
    ("latsum_ctx_comm_info", _I, [_P, _P, _P]),
    ("latsum_ctx_set_profiling", _I, [_P, _I]),
    ("latsum_ctx_profile", _I64, [_P, ctypes.c_char_p, _I64]),
    ("latsum_build_quadrature", _I, [_I, _D, _I, _D, _D, _D, _P, _P]),
    ("latsum_default_step_constant", _D, [_I, _D, _I, _D, _D, _I]),
    ("latsum_reference_shell", None, [_P, _P, _P]),
    ("latsum_verify_probes", None, [ctypes.c_uint64, _P, _I64, _P]),
    ("latsum_reference_build", _I, [_P, _I, _D, _P, _P, _I, _D, _P]),
    ("latsum_reference_destroy", None, [_P]),
    ("latsum_reference_info", _I, [_P, _P, _P, _P]),
    ("latsum_reference_factor", _I, [_P, _P, _I, _P]),
    ("latsum_reference_weights", _I, [_P, _P]),
    ("latsum_reference_quadrature", _I, [_P, _P, _P]),
    ("latsum_canonical_assemble", _I, [_P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P]),
    ("latsum_canonical_assemble_blocks", _I, [_P, _P, _I64, _P, _P, _P, _P]),
    ("latsum_canonical_destroy", None, [_P]),
    ("latsum_canonical_info", _I, [_P, _P, _P, _P, _P]),
    ("latsum_canonical_weights", _I, [_P, _P]),
    ("latsum_canonical_factor", _I, [_P, _P, _I, _P]),
    ("latsum_canonical_factor_device", _I, [_P, _P, _I, _P]),
    ("latsum_canonical_entries", _I, [_P, _P, _P, _I64, _P]),
    ("latsum_canonical_norm", _I, [_P, _P, _P]),
    ("latsum_canonical_eval_box_device", _I, [_P, _P, _P, _P, _P]),
    ("latsum_rhosvd", _I, [_P, _P, _P, _D, _I, _P, _P]),
    ("latsum_rhosvd_ex", _I, [_P, _P, _P, _D, _I, _I, _P, _P]),
    ("latsum_canonical_to_tucker", _I, [_P, _P, _P, _D, _I, _D, _P, _P, _P]),
    ("latsum_tucker_destroy", None, [_P]),
    ("latsum_tucker_has_core", _I, [_P]),
    ("latsum_tucker_info", _I, [_P, _P, _P]),
    ("latsum_tucker_singular_values", _I, [_P, _I, _P]),
    ("latsum_tucker_core_slab", _I, [_P, _P, _P, _P, _P]),
    ("latsum_tucker_core", _I, [_P, _P, _P]),
    ("latsum_tucker_factor", _I, [_P, _P, _I, _P]),
    ("latsum_format_spectral_report", _I64, [_P, _P, _P, _I64]),
    ("latsum_format_provenance", _I64, [_P, _P, _I64]),
    ("latsum_tucker_projected_form", _I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("latsum_tucker_entries", _I, [_P, _P, _P, _I64, _P]),
    ("latsum_tucker_eval_box", _I, [_P, _P, _P, _P, _P]),
    ("latsum_tucker_eval_box_device", _I, [_P, _P, _P, _P, _P]),
    ("latsum_sum_to_tucker", _I, [_P, _I, _D, _P, _P, _I, _D, _I64, _P, _P, _P, _I64, _P, _P,
                                  _D, _P, _P]),
    ("latsum_verify_entries", _I, [_P, _P, _I64, _P, _P, _P, _I64, _P]),
    ("latsum_canonical_from_host", _I, [_P, _P, _I64, _P, _P, _P, _P, _P]),
    ("latsum_canonical_concat", _I, [_P, _P, _P, _P]),
    ("latsum_ctx_set_accumulation", _I, [_P, _I]),
    ("latsum_tensor_write", _I, [_P, _P, _P, ctypes.c_char_p]),
    ("latsum_tensor_read", _I, [_P, ctypes.c_char_p, _P, _P]),
    ("latsum_dgemm_device", _I, [_P, _I, _I, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P,
                                 _I64]),
    ("latsum_sytrd_device", _I, [_P, _I64, _P, _I64, _P, _P, _P]),
    ("latsum_eig_sym_device", _I, [_P, _I64, _P, _I64, _P, _P, _I]),
    ("latsum_dgemm_ozaki_device", _I, [_P, _I, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64]),
]

_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", CSRC])
    else:
        subprocess.check_call(["make", "-s", "-C", CSRC], stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {CSRC}` "
                "(there is no CPU fallback for the lattice-sum path)")
        # LATSUM_LIBRARY: an instrumented build of the same sources (dev tools only)
        L = ctypes.CDLL(os.environ.get("LATSUM_LIBRARY", LIB_PATH))
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, ctx=None):
    if status == OK:
        return
    msg = lib().latsum_last_error(ctx).decode() if ctx else f"status {status}"
    if status == 2:
        raise WindowOverflowError(msg)
    raise ERRORS.get(status, RuntimeError)(msg)
