"""ctypes binding of libphylograd_b200.so (the C-ABI in include/phylograd_b200.h).

The product path has no CPU fallback: importing this module on a machine
without the built library raises, and every compute call runs CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "_build", "libphylograd_b200.so")

PG_OK = 0
PG_ERR_INVALID_ARGUMENT = 1
PG_ERR_RUNTIME = 2
PG_ERR_LOGIC = 3
PG_ERR_NEWICK = 4
PG_ERR_CUDA = 5
PG_ERR_NOT_SUPPORTED = 6
PG_ERR_NCCL = 7
REDUCE_NCCL = 0
REDUCE_FIXED_ORDER = 1

EVAL_LOGL = 1
EVAL_GRAD = 2
EVAL_HESS = 4
EVAL_RATE_GRAD = 8
EVAL_FORCE = 16
EVAL_POST_PASS = 32
EVAL_REQUIRE_POST = 64

# Every symbol include/phylograd_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "pg_default_options", "pg_last_error", "pg_create", "pg_destroy", "pg_set_topology", "pg_set_patterns",
    "pg_set_model", "pg_set_branch_generator", "pg_set_categories", "pg_set_branch_lengths",
    "pg_set_branch_lengths_device", "pg_get_branch_lengths", "pg_set_clock_durations", "pg_evaluate",
    "pg_evaluate_device", "pg_check_errors", "pg_set_stream", "pg_get_partials", "pg_get_site_log_likelihoods",
    "pg_node_visits", "pg_reset_node_visits", "pg_invalidate_caches", "pg_engine_info", "pg_last_walk_ms",
    "pg_timing", "pg_engine_variant",
    "pg_create_multi", "pg_group_info", "pg_clock_gradient",
    "pg_newick_parse", "pg_compress_codes", "pg_compress_result", "pg_compress_free", "pg_compress_codes_gpu",
    "pg_compress_result_gpu", "pg_compress_free_gpu", "pg_simulate_states_gpu", "pg_discrete_gamma",
]


class PgError(Exception):
    """Base class; subclasses mirror the reference's exception types."""


class InvalidArgument(PgError, ValueError):
    """std::invalid_argument in the reference."""


class RuntimeFailure(PgError, RuntimeError):
    """std::runtime_error in the reference (underflow / non-finite partials)."""


class LogicError(PgError):
    """std::logic_error in the reference (pass ordering)."""


class NewickError(PgError, RuntimeError):
    """phylograd::NewickError (tree.hpp:141-146); .position is the byte offset."""

    def __init__(self, msg):
        super().__init__(msg)
        import re

        m = re.search(r"\(at position (\d+)\)", msg)
        self.position = int(m.group(1)) if m else -1


class CudaFailure(PgError, RuntimeError):
    pass


class NotSupported(PgError, NotImplementedError):
    pass


class NcclFailure(PgError, RuntimeError):
    pass


_ERRORS = {
    PG_ERR_INVALID_ARGUMENT: InvalidArgument,
    PG_ERR_RUNTIME: RuntimeFailure,
    PG_ERR_LOGIC: LogicError,
    PG_ERR_NEWICK: NewickError,
    PG_ERR_CUDA: CudaFailure,
    PG_ERR_NOT_SUPPORTED: NotSupported,
    PG_ERR_NCCL: NcclFailure,
}


class Options(C.Structure):
    _fields_ = [
        ("rescaling_threshold", C.c_double),
        ("force_rescaling", C.c_int),
        ("disable_rescaling", C.c_int),
        ("device", C.c_int),
        ("capture_partials", C.c_int),
        ("reserved", C.c_int * 8),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"phylograd-b200: {SO_PATH} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(SO_PATH)
        _declare(L)
        _lib = L
    return _lib


P = C.c_void_p
I = C.c_int
D = C.c_double
PD = C.POINTER(C.c_double)
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)
PI8 = C.POINTER(C.c_int8)


def _declare(L):
    sig = {
        "pg_default_options": (None, [C.POINTER(Options)]),
        "pg_last_error": (C.c_char_p, []),
        "pg_create": (I, [C.POINTER(Options), C.POINTER(P)]),
        "pg_destroy": (None, [P]),
        "pg_set_topology": (I, [P, I, PI32, PI32, PI32]),
        "pg_set_patterns": (I, [P, I, I, PI8, I, PD, PI64]),
        "pg_set_model": (I, [P, I, PD, PD, I]),
        "pg_set_branch_generator": (I, [P, I, PD]),
        "pg_set_categories": (I, [P, I, PD, PD]),
        "pg_set_branch_lengths": (I, [P, PD]),
        "pg_set_branch_lengths_device": (I, [P, P]),
        "pg_get_branch_lengths": (I, [P, PD]),
        "pg_set_clock_durations": (I, [P, PD]),
        "pg_evaluate": (I, [P, I, PD, PD, PD]),
        "pg_evaluate_device": (I, [P, I, P]),
        "pg_check_errors": (I, [P]),
        "pg_set_stream": (I, [P, P]),
        "pg_get_partials": (I, [P, I, I, PD, PD, PD, PD]),
        "pg_get_site_log_likelihoods": (I, [P, PD]),
        "pg_node_visits": (C.c_uint64, [P]),
        "pg_reset_node_visits": (None, [P]),
        "pg_invalidate_caches": (None, [P]),
        "pg_engine_info": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
        "pg_last_walk_ms": (I, [P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
        "pg_timing": (I, [P, I, C.POINTER(I), C.POINTER(D), C.POINTER(D)]),
        "pg_engine_variant": (I, [P]),
        "pg_create_multi": (I, [C.POINTER(Options), I, C.POINTER(I), I, C.POINTER(P)]),
        "pg_group_info": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I)]),
        "pg_clock_gradient": (I, [P, PD, PD, PD, PD, PD]),
        "pg_newick_parse": (I, [C.c_char_p, C.POINTER(I), PI32, PI32, PD, PI32, C.c_char_p, C.c_int64]),
        "pg_compress_codes": (I, [I, C.c_int64, PI32, I, C.POINTER(P), C.POINTER(I)]),
        "pg_compress_result": (I, [P, PI32, PI64, PI32]),
        "pg_compress_free": (None, [P]),
        "pg_compress_codes_gpu": (I, [I, C.c_int64, P, I, I, I, C.POINTER(P), C.POINTER(I)]),
        "pg_compress_result_gpu": (I, [P, P, PI64, PI32, C.POINTER(C.c_float)]),
        "pg_compress_free_gpu": (None, [P]),
        "pg_simulate_states_gpu": (I, [I, PI32, PI32, I, PD, PD, I, I, PD, PD, PD, C.c_int64, C.c_uint64, D, I, P, I,
                                       C.POINTER(C.c_float)]),
        "pg_discrete_gamma": (I, [D, I, PD, PD]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def check(rc: int):
    if rc == PG_OK:
        return
    msg = lib().pg_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, PgError)(msg)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
