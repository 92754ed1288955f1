"""ctypes binding of the C-ABI in include/pbbgpu.h (libpbbgpu.so, built in-tree).

The shared library is the product: there is no Python or CPU fallback for any compute
entry point. If the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBBGPU_LIB") or os.path.join(_HERE, "libpbbgpu.so")  # override: A/B dev runs

PBBGPU_OK = 0
PBBGPU_ERR_ARG = -1
PBBGPU_ERR_STATE = -2
PBBGPU_ERR_CUDA = -3
PBBGPU_ERR_CAPACITY = -4
PBBGPU_ERR_TRANSPORT = -5
LB1 = 1
LB2 = 2

# every symbol include/pbbgpu.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "pbbgpu_last_error", "pbbgpu_device_count", "pbbgpu_taillard", "pbbgpu_taillard_named",
    "pbbgpu_makespan", "pbbgpu_neh", "pbbgpu_create", "pbbgpu_destroy", "pbbgpu_load_instance", "pbbgpu_seed", "pbbgpu_K",
    "pbbgpu_set_initial_bound", "pbbgpu_assign", "pbbgpu_assign_split", "pbbgpu_run_round",
    "pbbgpu_active_count", "pbbgpu_snapshot", "pbbgpu_best", "pbbgpu_offer_bound",
    "pbbgpu_stats", "pbbgpu_histogram", "pbbgpu_decompose_batch", "pbbgpu_solve", "pbbgpu_int32_peak",
    "pbbgpu_assign_split_range", "pbbgpu_export", "pbbgpu_debug_state", "pbbgpu_assign_split_strided",
    "pbbgpu_insertion_ls", "pbbgpu_offer_schedule", "pbbgpu_promote", "pbbgpu_explorer_lengths",
    "pbbgpu_best_schedule", "pbbgpu_snapshot_ex", "pbbgpu_apply_work_update", "pbbgpu_improved_since_mark",
    "pbbgpu_steals_since_mark", "pbbgpu_reset_steal_mark", "pbbgpu_take_census", "pbbgpu_flush_timeline",
    "pbbgpu_group_handle_size", "pbbgpu_group_create", "pbbgpu_group_open", "pbbgpu_group_reset",
    "pbbgpu_group_solve", "pbbgpu_group_close", "pbbgpu_pool_shape", "pbbgpu_pool_times", "pbbgpu_worker_run",
    "pbbgpu_wire_reencode",
)


class Config(ctypes.Structure):
    _fields_ = [
        ("explorers", ctypes.c_int),
        ("group", ctypes.c_int),
        ("steps_per_round", ctypes.c_int),
        ("disable_pruning", ctypes.c_int),
        ("pinned", ctypes.c_int),
        ("time_limit_s", ctypes.c_double),
        ("min_steal_log2", ctypes.c_double),
        ("device", ctypes.c_int),
        ("block", ctypes.c_int),
        ("round_us", ctypes.c_double),
        ("steal_trigger", ctypes.c_double),
        ("rounds_per_sync", ctypes.c_int),
        ("max_split", ctypes.c_int),
        ("split_mode", ctypes.c_int),
        ("steal_policy", ctypes.c_int),
        ("record_census", ctypes.c_int),
        ("census_cap", ctypes.c_int),
        ("timeline_path", ctypes.c_char_p),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("decomposed", ctypes.c_uint64),
        ("unique", ctypes.c_uint64),
        ("replay_dups", ctypes.c_uint64),
        ("leaves", ctypes.c_uint64),
        ("improvements", ctypes.c_uint64),
        ("local_steals", ctypes.c_uint64),
        ("steal_phases", ctypes.c_uint64),
        ("intervals_initialized", ctypes.c_uint64),
        ("rounds", ctypes.c_uint64),
        ("steps", ctypes.c_uint64),
        ("wall_s", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("completed", ctypes.c_int),
        ("K", ctypes.c_int),
        ("group", ctypes.c_int),
        ("steps_per_round", ctypes.c_int),
        ("device_ms", ctypes.c_double),
        ("kernel_launches", ctypes.c_uint64),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("block", ctypes.c_int),
        ("batch_kernel_ms", ctypes.c_double),
        ("steal_kernel_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class GroupStats(ctypes.Structure):
    _fields_ = [
        ("syncs", ctypes.c_uint64),
        ("exchanges", ctypes.c_uint64),
        ("imported", ctypes.c_uint64),
        ("exported", ctypes.c_uint64),
        ("wall_s", ctypes.c_double),
        ("device_ms", ctypes.c_double),
        ("completed", ctypes.c_int),
        ("exchange_us_per_round", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class WorkerConfig(ctypes.Structure):
    _fields_ = [
        ("worker_id", ctypes.c_uint32),
        ("checkpoint_period_s", ctypes.c_double),
        ("initial_ub", ctypes.c_int64),
        ("rng_seed", ctypes.c_uint64),
        ("ils_iterations", ctypes.c_int),
        ("send_initial_best", ctypes.c_int),
    ]


class WorkerResult(ctypes.Structure):
    _fields_ = [
        ("local_best", ctypes.c_int64),
        ("has_schedule", ctypes.c_int),
        ("checkpoints_sent", ctypes.c_uint64),
        ("bests_sent", ctypes.c_uint64),
        ("updates_applied", ctypes.c_uint64),
        ("messages", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load libpbbgpu.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the product has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i32p = ctypes.POINTER(ctypes.c_int32)
    i64p = ctypes.POINTER(ctypes.c_int64)
    u16p = ctypes.POINTER(ctypes.c_uint16)
    u8p = ctypes.POINTER(ctypes.c_uint8)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    ip = ctypes.POINTER(ctypes.c_int)
    sig = {
        "pbbgpu_last_error": (ctypes.c_char_p, []),
        "pbbgpu_device_count": (ctypes.c_int, []),
        "pbbgpu_taillard": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int32, i32p]),
        "pbbgpu_taillard_named": (ctypes.c_int, [ctypes.c_char_p, ip, ip, i32p]),
        "pbbgpu_makespan": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, i32p, i32p]),
        "pbbgpu_neh": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, i32p, i32p]),
        "pbbgpu_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int,
                                         ctypes.POINTER(Config), ctypes.POINTER(P)]),
        "pbbgpu_destroy": (None, [P]),
        "pbbgpu_load_instance": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int32)]),
        "pbbgpu_seed": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "pbbgpu_K": (ctypes.c_int, [P]),
        "pbbgpu_set_initial_bound": (ctypes.c_int, [P, ctypes.c_int64, i32p, ctypes.c_int]),
        "pbbgpu_assign": (ctypes.c_int, [P, u16p, u16p, u8p, ctypes.c_int]),
        "pbbgpu_assign_split": (ctypes.c_int, [P, ctypes.c_int]),
        "pbbgpu_run_round": (ctypes.c_int, [P, ip]),
        "pbbgpu_active_count": (ctypes.c_int, [P, ip]),
        "pbbgpu_snapshot": (ctypes.c_int, [P, u16p, u16p, u8p, ctypes.c_int, ip]),
        "pbbgpu_best": (ctypes.c_int, [P, i64p, i32p, ip]),
        "pbbgpu_best_schedule": (ctypes.c_int, [P, i64p, i32p, ip]),
        "pbbgpu_snapshot_ex": (ctypes.c_int, [P, u16p, u16p, u8p, ctypes.c_int, ip, u64p]),
        "pbbgpu_apply_work_update": (ctypes.c_int, [P, u16p, u16p, u8p, ctypes.c_int]),
        "pbbgpu_improved_since_mark": (ctypes.c_int, [P, ip]),
        "pbbgpu_steals_since_mark": (ctypes.c_int, [P, u64p]),
        "pbbgpu_reset_steal_mark": (ctypes.c_int, [P]),
        "pbbgpu_take_census": (ctypes.c_int, [P, u64p, ctypes.c_int64, i64p]),
        "pbbgpu_flush_timeline": (ctypes.c_int, [P]),
        "pbbgpu_group_handle_size": (ctypes.c_int, []),
        "pbbgpu_group_create": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
        "pbbgpu_group_open": (ctypes.c_int, [P, ctypes.c_void_p]),
        "pbbgpu_group_reset": (ctypes.c_int, [P]),
        "pbbgpu_group_solve": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                              ctypes.POINTER(GroupStats)]),
        "pbbgpu_group_close": (ctypes.c_int, [P]),
        "pbbgpu_pool_shape": (ctypes.c_int, [P, ip, ip]),
        "pbbgpu_pool_times": (ctypes.c_int, [P, i32p]),
        "pbbgpu_worker_run": (ctypes.c_int, [P, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(WorkerConfig),
                                             ctypes.POINTER(WorkerResult)]),
        "pbbgpu_wire_reencode": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_void_p, ctypes.c_int64, i64p]),
        "pbbgpu_offer_bound": (ctypes.c_int, [P, ctypes.c_int64]),
        "pbbgpu_stats": (ctypes.c_int, [P, ctypes.POINTER(Stats)]),
        "pbbgpu_histogram": (ctypes.c_int, [P, u64p, ctypes.c_int]),
        "pbbgpu_decompose_batch": (ctypes.c_int, [P, i32p, i32p, i32p, ctypes.c_int, ctypes.c_int64,
                                                  i64p, u8p, u8p, i64p, i64p]),
        "pbbgpu_assign_split_range": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "pbbgpu_assign_split_strided": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "pbbgpu_export": (ctypes.c_int, [P, ctypes.c_int, u16p, u16p, u8p, ip]),
        "pbbgpu_debug_state": (ctypes.c_int, [P, u8p, ctypes.c_int64, ip, ip]),
        "pbbgpu_insertion_ls": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, i32p, i32p, ctypes.c_uint64,
                                                 ctypes.c_double, ctypes.c_uint64, i32p]),
        "pbbgpu_offer_schedule": (ctypes.c_int, [P, i32p, ctypes.c_int64, ip]),
        "pbbgpu_promote": (ctypes.c_int, [P, ctypes.c_int, i32p, i64p, ip]),
        "pbbgpu_explorer_lengths": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_float), ctypes.c_int]),
        "pbbgpu_int32_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
        "pbbgpu_solve": (ctypes.c_int, [P, ctypes.c_int64, u16p, u16p, u8p, ctypes.c_int, i64p, i32p,
                                        ip, ctypes.POINTER(Stats)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class PbbError(RuntimeError):
    """Error returned through the C-ABI (status code + pbbgpu_last_error())."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"pbbgpu error {code}: {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != PBBGPU_OK:
        msg = load().pbbgpu_last_error()
        msg = msg.decode() if msg else ""
        if rc == PBBGPU_ERR_ARG:
            raise ValueError(msg)
        raise PbbError(rc, msg)
