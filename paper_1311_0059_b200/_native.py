"""ctypes binding of libaggb200.so (include/aggb200.h).

The library is built in-tree (``paper_1311_0059_b200/lib/libaggb200.so``) by
``paper_1311_0059_b200.build`` / ``__graft_entry__.build()``.  There is no CPU
fallback: if the library is missing every entry point raises
``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AGGB_LIB_OVERRIDE") or os.path.join(HERE, "lib", "libaggb200.so")  # (experiment builds)
HEADER = os.path.join(os.path.dirname(HERE), "include", "aggb200.h")

AGGB_OK = 0
AGGB_INVALID_BUDGET = 1
AGGB_BUDGET_EXHAUSTED = 2
AGGB_CAPACITY_EXCEEDED = 3
AGGB_SPEC_ERROR = 4
AGGB_ORDER_ERROR = 5
AGGB_CUDA_ERROR = 6
AGGB_INVALID_ARG = 7
AGGB_INVALID_RECORD = 8

ALGO = {"sort_based": 0, "hash_sort": 1, "original_hh": 2, "shared_hash": 3,
        "dynamic_destaging": 4, "pre_partitioning": 5}
FN = {"sum": 0, "count": 1, "avg": 2, "min": 3, "max": 4}
I64, F64, I32 = 0, 1, 2
INPUT_RAW, INPUT_STATES = 0, 1
MAX_FNS, MAX_VALS, MAX_KEYS = 32, 32, 2

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = ("aggb_create", "aggb_push", "aggb_finish", "aggb_copy_result",
           "aggb_exchange_record_bytes", "aggb_exchange_pack", "aggb_push_partials",
           "aggb_exchange_raw_record_bytes", "aggb_exchange_pack_raw", "aggb_pool_host_bytes",
           "aggb_metrics_get", "aggb_reset", "aggb_destroy", "aggb_last_error",
           "aggb_generate", "aggb_l2_flush", "aggb_version", "aggb_profile",
           "aggb_kernel_stats")


class NativeLibraryMissing(RuntimeError):
    """The CUDA library is not built; the GPU path has no fallback."""


class Config(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("memory_frames", ctypes.c_int32),
                ("frame_size", ctypes.c_int32), ("input_sorted", ctypes.c_int32),
                ("budget_groups", ctypes.c_int64), ("fudge", ctypes.c_double),
                ("slot_ratio", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("group_estimate", ctypes.c_double), ("stats_R", ctypes.c_double),
                ("stats_R_t", ctypes.c_double), ("stats_G", ctypes.c_double),
                ("stats_G_t", ctypes.c_double), ("level", ctypes.c_int32),
                ("emit_partials", ctypes.c_int32), ("reserved_", ctypes.c_int32 * 6)]


class Spec(ctypes.Structure):
    _fields_ = [("n_fns", ctypes.c_int32), ("fn", ctypes.c_int32 * MAX_FNS),
                ("col", ctypes.c_int32 * MAX_FNS), ("n_keys", ctypes.c_int32),
                ("key_type", ctypes.c_int32 * MAX_KEYS), ("n_vals", ctypes.c_int32),
                ("val_type", ctypes.c_int32 * MAX_VALS), ("input_kind", ctypes.c_int32)]


class Input(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("key", ctypes.c_void_p * MAX_KEYS),
                ("key_stride", ctypes.c_int64 * MAX_KEYS), ("val", ctypes.c_void_p * MAX_VALS),
                ("val_stride", ctypes.c_int64 * MAX_VALS), ("on_host", ctypes.c_int32),
                ("reserved_", ctypes.c_int32)]


class Result(ctypes.Structure):
    _fields_ = [("n_groups", ctypes.c_int64), ("key", ctypes.c_void_p * MAX_KEYS),
                ("out", ctypes.c_void_p * MAX_FNS), ("out_type", ctypes.c_int32 * MAX_FNS),
                ("sorted", ctypes.c_int32), ("reserved_", ctypes.c_int32)]


class Metrics(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "records", "output_groups", "resident_groups", "spilled_records", "spilled_bytes",
        "spilled_partitions", "recursion_depth", "grace_levels", "fallbacks",
        "high_water_bytes", "budget_groups", "partitions_level0", "kernel_launches",
        "hbm_bytes_alg", "level0_spilled_records", "child_subpasses")]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.aggb_create.argtypes = [i32, ctypes.POINTER(Config), ctypes.POINTER(Spec), vp,
                              ctypes.POINTER(vp)]
    L.aggb_push.argtypes = [vp, ctypes.POINTER(Input)]
    L.aggb_finish.argtypes = [vp, ctypes.POINTER(Result)]
    L.aggb_copy_result.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.aggb_exchange_record_bytes.argtypes = [vp]
    L.aggb_exchange_record_bytes.restype = i64
    L.aggb_exchange_pack.argtypes = [vp, i32, vp, ctypes.POINTER(i64)]
    L.aggb_push_partials.argtypes = [vp, vp, i64]
    L.aggb_exchange_raw_record_bytes.argtypes = [vp]
    L.aggb_exchange_raw_record_bytes.restype = i64
    L.aggb_pool_host_bytes.argtypes = [vp]
    L.aggb_pool_host_bytes.restype = i64
    L.aggb_exchange_pack_raw.argtypes = [vp, ctypes.POINTER(Input), i32, vp, ctypes.POINTER(i64)]
    L.aggb_metrics_get.argtypes = [vp, ctypes.POINTER(Metrics)]
    L.aggb_reset.argtypes = [vp]
    L.aggb_destroy.argtypes = [vp]
    L.aggb_destroy.restype = None
    L.aggb_last_error.restype = ctypes.c_char_p
    L.aggb_version.restype = ctypes.c_char_p
    L.aggb_generate.argtypes = [vp, i32, ctypes.c_uint64, ctypes.c_uint64, i64, i64, i64, i64,
                                vp, i64, ctypes.c_uint64, ctypes.c_uint64, vp, i64]
    L.aggb_l2_flush.argtypes = [vp, vp, i64]
    L.aggb_profile.argtypes = [vp, i32]
    L.aggb_kernel_stats.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_char_p),
                                    ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]
    for name in ("aggb_create", "aggb_push", "aggb_finish", "aggb_copy_result",
                 "aggb_exchange_pack", "aggb_push_partials", "aggb_exchange_pack_raw",
                 "aggb_metrics_get", "aggb_reset",
                 "aggb_generate", "aggb_l2_flush", "aggb_profile", "aggb_kernel_stats"):
        getattr(L, name).restype = i32
    _lib = L
    return L


def last_error() -> str:
    return (load().aggb_last_error() or b"").decode()


def check(status: int, what: str = "") -> None:
    """Map a status onto the reference's exception classes (core.py:28-61)."""
    if status == AGGB_OK:
        return
    from paper_1311_0059_b200 import core
    msg = f"{what}: {last_error()}" if what else last_error()
    cls = {AGGB_INVALID_BUDGET: core.InvalidBudget,
           AGGB_BUDGET_EXHAUSTED: core.BudgetExhausted,
           AGGB_CAPACITY_EXCEEDED: core.CapacityExceeded,
           AGGB_SPEC_ERROR: core.SpecError,
           AGGB_ORDER_ERROR: core.MergeOrderError,
           AGGB_INVALID_RECORD: core.InvalidRecord}.get(status, core.AggregationError)
    raise cls(msg)
