"""ctypes binding of the C ABI in include/ss_b200.h.

This module is the only place that talks to libss_b200.so.  It fails
loudly when the library is missing: there is no CPU fallback anywhere in
the package.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ExecutionError, raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SS_B200_LIB") or os.path.join(HERE, "_lib", "libss_b200.so")

AGG_COUNT, AGG_SUM, AGG_AVG, AGG_MIN, AGG_MAX = 1, 2, 4, 8, 16
POLICY_CODES = {"no": 0, "first": 1, "all": 2, "prob": 3, "best": 4,
                "shift": 5, "shiftlocal": 6}
FRONT_CODE, BACK_CODE = 0, 1


class Config(C.Structure):
    _fields_ = [("n_groups", C.c_int64), ("window", C.c_int64),
                ("n_partitions", C.c_int32), ("key_bits", C.c_int32),
                ("agg_mask", C.c_uint32), ("scope", C.c_int32),
                ("device", C.c_int32), ("reserved", C.c_int32),
                ("max_batch", C.c_int64), ("sub_batch", C.c_int64),
                ("pool_values", C.c_int64)]


class Balancer(C.Structure):
    _fields_ = [("policy", C.c_int32), ("reserved", C.c_int32),
                ("thread_threshold", C.c_int64), ("pot", C.c_double),
                ("max_moves", C.c_int64), ("split", C.c_int32),
                ("split_max", C.c_int32), ("split_target", C.c_double)]


class MoveC(C.Structure):
    _fields_ = [("group", C.c_int32), ("src", C.c_int32),
                ("dst", C.c_int32), ("placement", C.c_int32)]


class StepReport(C.Structure):
    _fields_ = [("tuples", C.c_int64), ("imbalance", C.c_int64),
                ("moves", C.c_int64), ("moves_applied_before", C.c_int64),
                ("scanned", C.c_int64), ("max_load", C.c_int64),
                ("touched", C.c_int64), ("split_groups", C.c_int64),
                ("mean_load", C.c_double), ("load_ratio", C.c_double)]


_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "ss_version": (C.c_char_p, []),
    "ss_launch_count": (C.c_longlong, [C.c_int]),
    "ss_sub_batch": (C.c_longlong, [_P]),
    "ss_set_host_emit": (C.c_int, [_P, C.c_int]),
    "ss_set_graphs": (C.c_int, [_P, C.c_int]),
    "ss_results_pull": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, C.POINTER(C.c_int64)]),
    "ss_create": (C.c_int, [C.POINTER(Config), C.POINTER(_P)]),
    "ss_destroy": (None, [_P]),
    "ss_set_stream": (C.c_int, [_P, _P]),
    "ss_sync": (C.c_int, [_P]),
    "ss_last_error": (C.c_char_p, [_P]),
    "ss_set_assignment": (C.c_int, [_P, _P, _P]),
    "ss_get_assignment": (C.c_int, [_P, _P, _P, _P]),
    "ss_apply_moves": (C.c_int, [_P, _P, _I64]),
    "ss_count": (C.c_int, [_P, _P, _I64, _P, _P]),
    "ss_reorder": (C.c_int, [_P, _P, _P, _I64, _P, _P, _P]),
    "ss_ingest": (C.c_int, [_P, _P, _P, _I64]),
    "ss_balance": (C.c_int, [_P, _P, _I64, C.POINTER(Balancer), _P, _P, _P, _P]),
    "ss_step": (C.c_int, [_P, _P, _P, _I64, C.POINTER(Balancer), C.POINTER(StepReport)]),
    "ss_last_report": (C.c_int, [_P, C.POINTER(StepReport)]),
    "ss_last_loads": (C.c_int, [_P, _P]),
    "ss_last_moves": (C.c_int, [_P, _P, _I64, _P]),
    "ss_last_part_ns": (C.c_int, [_P, _P]),
    "ss_last_part_work": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "ss_snapshot": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "ss_export_values": (C.c_int, [_P, _I64, _P, _I64, _P]),
    "ss_results": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "ss_profile": (C.c_int, [_P, C.c_int]),
    "ss_profile_read": (C.c_int, [_P, _P, _P, C.c_int]),
    "ss_alg_bytes": (C.c_int, [_P, _P, C.c_int]),
    "ss_results_raw": (C.c_int, [_P, _I64, _P, _P, _P]),
    "ss_set_owner": (C.c_int, [_P, _P, C.c_int]),
    "ss_route": (C.c_int, [_P, _P, _P, _I64, _P, _P, _P]),
    "ss_group_counts": (C.c_int, [_P, _P]),
    "ss_balance_counts": (C.c_int, [_P, _P, C.POINTER(Balancer), _P, _P, _P, _P]),
    "ss_export_state": (C.c_int, [_P, _P, _I64, _P, _P, _I64, _P]),
    "ss_import_state": (C.c_int, [_P, _P, _I64, _P, _P]),
    "ss_route_records": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "ss_set_owner_dev": (C.c_int, [_P, _P, C.c_int]),
    "ss_balance_apply_dev": (C.c_int, [_P, _P, C.POINTER(Balancer), _P, _P, _P]),
    "ss_export_moves_dev": (C.c_int, [_P, _P, _P, C.c_int, _P, _I64, _P]),
    "ss_import_blob_dev": (C.c_int, [_P, _P, _P, C.c_int, C.c_int]),
    "ss_set_bucket_owner": (C.c_int, [_P, _P, C.c_int]),
    "ss_route_records64": (C.c_int, [_P, _P, _P, _I64, _P, _P]),
    "ss_step_records64": (C.c_int, [_P, _P, C.c_int64, C.POINTER(Balancer), C.POINTER(StepReport)]),
    "ss_bucket_counts_dev": (C.c_int, [_P, _P]),
    "ss_export_moves64_dev": (C.c_int, [_P, _P, _P, C.c_int, _P, _I64, _P]),
    "ss_import_blob64_dev": (C.c_int, [_P, _P, _P, C.c_int]),
    "ss_map_keys": (C.c_int, [_P, _P, _I64, _P]),
    "ss_set_trace": (C.c_int, [_P, C.c_int]),
    "ss_trace": (C.c_int, [_P, C.c_int64, _P, _P, C.POINTER(C.c_int64)]),
    "ss_step_records": (C.c_int, [_P, _P, C.c_int64, C.POINTER(Balancer), C.POINTER(StepReport)]),
    "ss_step_keys64": (C.c_int, [_P, _P, _P, _I64, C.POINTER(Balancer), C.POINTER(StepReport)]),
    "ss_slot_keys": (C.c_int, [_P, _P, _P]),
    "ss_set_key_pipeline": (C.c_int, [_P, C.c_int]),
}
KERNEL_CLASSES = ("count", "stats", "place", "ingest", "emit", "apply", "balance")
EXPORTS = tuple(_SIGS)

_lib = None


def load():
    """Load libss_b200.so (raises ExecutionError when it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExecutionError(
            f"CUDA engine library missing: {LIB_PATH} (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(handle, rc: int) -> None:
    if rc:
        msg = load().ss_last_error(handle)
        raise_for_status(rc, msg.decode() if msg else f"status {rc}")
