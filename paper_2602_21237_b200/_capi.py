"""ctypes binding of librelab_b200.so (the C ABI in include/relab_b200.h).

The reference tensor path is Python calling numpy; its B200 replacement is
Python calling this library. There is deliberately no fallback: if the
library is missing the import of the operators fails loudly, and every
compute entry point requires CUDA device pointers.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import DeviceError, OutputTooLarge

LIB_NAME = "librelab_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

RL_OK = 0
RL_ERR_BAD_ARG = 1
RL_ERR_OUTPUT_TOO_LARGE = 2
RL_ERR_WORKSPACE = 3
RL_ERR_TOO_MANY_ROWS = 4
RL_ERR_IO = 5
RL_ERR_CUDA = 1000

RL_COL_INT64 = 0
RL_COL_BYTES = 1
RL_SIDE_LEFT = 0
RL_SIDE_RIGHT = 1
RL_SIDE_KEY = 2
RL_MAX_COLUMNS = 32
RL_MAX_ROWS = 2**32 - 1
RL_SORT_EVENTS = 3
RL_SORT_STAMPS = 12
RL_MAX_SPLIT_SAMPLES = 2048
RL_SORT_MAX_FUSED_COLUMNS = 8
RL_PUSH_MAX_PARTS = 64
RL_PUSH_MAX_COLUMNS = 8


class RlColumn(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_void_p),
        ("dst", ctypes.c_void_p),
        ("width", ctypes.c_int32),
        ("side", ctypes.c_int32),
    ]


class RlJoinPlan(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in (
        "scalars", "left_positions", "left_key_values", "left_offsets", "right_positions", "right_key_values",
        "right_offsets", "matched_keys", "left_starts", "left_counts", "right_starts", "right_counts",
        "pair_offsets")]


class RlBjoinPlan(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in (
        "rows_left", "rows_right", "sub_off_left", "sub_off_right", "flags_left", "flags_right", "counts",
        "offsets", "scalars", "left_keys")] + [("levels", ctypes.c_int32)] + [
        (name, ctypes.c_void_p) for name in ("pay_left", "pay_right")] + [
        ("words_left", ctypes.c_int32), ("words_right", ctypes.c_int32),
        ("carry_cols_left", ctypes.c_int32), ("carry_cols_right", ctypes.c_int32),
        ("carry_src_left", ctypes.c_void_p * 4), ("carry_src_right", ctypes.c_void_p * 4),
        ("carry_width_left", ctypes.c_int32 * 4), ("carry_width_right", ctypes.c_int32 * 4),
        ("carry_off_left", ctypes.c_int32 * 4), ("carry_off_right", ctypes.c_int32 * 4),
        ("sel_pairs", ctypes.c_void_p), ("sel_idx", ctypes.c_void_p), ("run_sel", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); every symbol declared in include/relab_b200.h
SIGNATURES = {
    "rl_abi_version": (ctypes.c_int, []),
    "rl_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "rl_device_sm_count": (ctypes.c_int, []),
    "rl_launch_count": (_I64, []),
    "rl_push_rows": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _I32, _P, _P, _P]),
    "rl_push_rows_gid": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _I32, _P, _P, _I64, _P]),
    "rl_sample_keys": (ctypes.c_int, [_P, _I64, _I32, _I64, _I32, _P, _P]),
    "rl_pick_splitters": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _P]),
    "rl_global_ids": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, _P]),
    "rl_stager_file_h2d": (ctypes.c_int, [_P, _P, _I32, ctypes.c_uint64, _SZ, _P, _P]),
    "rl_stager_file_d2h": (ctypes.c_int, [_P, _P, _I32, ctypes.c_uint64, _SZ, _P]),
    "rl_stager_file_read": (ctypes.c_int, [_P, _P, _I32, ctypes.c_uint64, _SZ]),
    "rl_sort_workspace_bytes": (_SZ, [_I64]),
    "rl_sort_axis": (ctypes.c_int, [_P, _I32, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _SZ, _P]),
    "rl_sort_axis_profiled": (
        ctypes.c_int,
        [_P, _I32, _I32, _I32, _I32, _P, _I64, _P, _P, ctypes.POINTER(RlColumn), _I32, _P, _SZ, _P,
         ctypes.POINTER(ctypes.c_void_p), _P],
    ),
    "rl_sort_axis_gather": (
        ctypes.c_int,
        [_P, _I32, _I32, _I32, _I32, _P, _I64, _P, _P, ctypes.POINTER(RlColumn), _I32, _P, _SZ, _P],
    ),
    "rl_sort_carry_workspace_bytes": (_SZ, [_I64, _I32]),
    "rl_sort_axis_carry": (ctypes.c_int, [_P, _I64, _I32, _P, _P, ctypes.POINTER(RlColumn), _I32, _P, _SZ, _P]),
    "rl_run_bounds_workspace_bytes": (_SZ, [_I64]),
    "rl_run_bounds": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "rl_align_workspace_bytes": (_SZ, [_I64]),
    "rl_key_axis_align": (
        ctypes.c_int,
        [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
    ),
    "rl_join_plan_workspace_bytes": (_SZ, [_I64, _I64]),
    "rl_join_plan_build": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _SZ, ctypes.POINTER(RlJoinPlan), _P]),
    "rl_join_expand": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _I64, _P, _P, _U64, _U64, _P, _P, ctypes.POINTER(RlColumn), _I32, _P],
    ),
    "rl_join_pair_checksum": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _P, _U64, _U64, _P, _P]),
    "rl_bjoin_workspace_bytes": (_SZ, [_I64, _I64, _I32, _I32]),
    "rl_bjoin_carry_words": (ctypes.c_int, [ctypes.POINTER(RlColumn), _I32]),
    "rl_bjoin_plan_build": (ctypes.c_int, [_P, _I64, _P, _I64, ctypes.POINTER(RlColumn), _I32,
                                           ctypes.POINTER(RlColumn), _I32, _P, _SZ, ctypes.POINTER(RlBjoinPlan), _P]),
    "rl_bjoin_expand": (ctypes.c_int, [ctypes.POINTER(RlBjoinPlan), _U64, _U64, _P, _P, ctypes.POINTER(RlColumn),
                                       _I32, _P]),
    "rl_bjoin_expand_strided": (ctypes.c_int, [ctypes.POINTER(RlBjoinPlan), _U64, _U64, _P, _P,
                                               ctypes.POINTER(RlColumn), _I32, _P, _P]),
    "rl_bjoin_pair_checksum": (ctypes.c_int, [ctypes.POINTER(RlBjoinPlan), _U64, _U64, _P, _P]),
    "rl_gather_rows_split16": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P]),
    "rl_gather_rows": (ctypes.c_int, [_P, _I64, ctypes.POINTER(RlColumn), _I32, _P]),
    "rl_widen_u32": (ctypes.c_int, [_P, _I64, _P, _P]),
    "rl_partition_workspace_bytes": (_SZ, [_I64, _I32]),
    "rl_range_partition": (
        ctypes.c_int,
        [_P, _I64, _I64, _P, _P, _I32, _I32, ctypes.POINTER(RlColumn), _I32, _P, _P, _P, _SZ, _P],
    ),
    "rl_multiset_digest": (ctypes.c_int, [ctypes.POINTER(RlColumn), _I32, _I64, _P, _P]),
    "rl_stager_create": (_P, [_I32, _SZ, _I32]),
    "rl_stager_destroy": (None, [_P]),
    "rl_stager_h2d": (ctypes.c_int, [_P, _P, _P, _SZ, _P, _P]),
    "rl_host_register": (ctypes.c_int, [_P, _SZ]),
    "rl_host_unregister": (ctypes.c_int, [_P]),
    "rl_host_is_pinned": (ctypes.c_int, [_P]),
    "rl_stager_h2d_pinned": (ctypes.c_int, [_P, _P, _P, _SZ, _P, _P]),
    "rl_stager_drain": (ctypes.c_int, [_P]),
    "rl_hash_partition": (
        ctypes.c_int,
        [_P, _I64, _I32, _U64, ctypes.POINTER(RlColumn), _I32, _P, _P, _P, _SZ, _P],
    ),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library. Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("RELAB_B200_LIB") or str(LIB_PATH)  # empty = unset
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 tensor path has no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rl_abi_version() != 1:
        raise ImportError(f"{path}: unexpected ABI version {lib.rl_abi_version()}")
    _lib = lib
    return lib


def strerror(status: int) -> str:
    return load().rl_strerror(status).decode()


def check(status: int, what: str) -> None:
    """Map a C status to the reference's exception classes."""
    if status == RL_OK:
        return
    msg = f"{what}: {strerror(status)} (status {status})"
    if status in (RL_ERR_BAD_ARG, RL_ERR_TOO_MANY_ROWS):
        raise ValueError(msg)
    if status == RL_ERR_OUTPUT_TOO_LARGE:
        raise OutputTooLarge(msg)
    if status == RL_ERR_IO:
        raise OSError(msg)
    raise DeviceError(msg)


def columns_array(cols) -> tuple:
    """(ctypes array, count) from an iterable of (src_ptr, dst_ptr, width, side)."""
    cols = list(cols)
    if len(cols) > RL_MAX_COLUMNS:
        raise ValueError(f"at most {RL_MAX_COLUMNS} columns per launch")
    arr = (RlColumn * max(1, len(cols)))()
    for i, (src, dst, width, side) in enumerate(cols):
        arr[i] = RlColumn(src or None, dst or None, int(width), int(side))
    return arr, len(cols)
