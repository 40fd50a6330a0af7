"""Host-side checks of the C ABI and the Python boundary (no GPU needed)."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2602_21237_b200 import _capi as C
from paper_2602_21237_b200 import records as R

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "relab_b200.h"


def declared_symbols():
    return sorted(set(re.findall(r"RL_API\s+[\w\s\*]+?\b(rl_\w+)\s*\(", HEADER.read_text())))


def test_library_loads_and_exports_every_declared_symbol():
    lib = C.load()
    names = declared_symbols()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
        assert name in C.SIGNATURES, f"{name} declared in the header but not typed in _capi"
    assert set(C.SIGNATURES) == set(names)


def test_abi_version_and_strerror():
    lib = C.load()
    assert lib.rl_abi_version() == 1
    assert C.strerror(0) == "ok"
    assert "cap" in C.strerror(C.RL_ERR_OUTPUT_TOO_LARGE)
    assert C.strerror(C.RL_ERR_CUDA + 2)  # cudaErrorMemoryAllocation text


def test_header_constants_match_python():
    text = HEADER.read_text()
    for name in ("RL_OK", "RL_ERR_BAD_ARG", "RL_ERR_OUTPUT_TOO_LARGE", "RL_ERR_WORKSPACE", "RL_ERR_TOO_MANY_ROWS",
                 "RL_ERR_CUDA", "RL_COL_INT64", "RL_COL_BYTES", "RL_SIDE_LEFT", "RL_SIDE_RIGHT", "RL_SIDE_KEY",
                 "RL_MAX_COLUMNS"):
        m = re.search(rf"#define {name} (\d+)", text)
        assert m and int(m.group(1)) == getattr(C, name), name


def test_workspace_queries_are_monotone():
    lib = C.load()
    prev = 0
    for n in (0, 1, 4095, 4096, 4097, 10**6, 10**8):
        ws = lib.rl_sort_workspace_bytes(n)
        assert ws >= prev
        assert ws >= 24 * n  # two key + two value ping-pong buffers
        prev = ws
    assert lib.rl_run_bounds_workspace_bytes(10**6) > 0
    assert lib.rl_align_workspace_bytes(10**6) > 0
    assert lib.rl_partition_workspace_bytes(10**6, 8) > lib.rl_sort_workspace_bytes(10**6)


def test_status_mapping():
    C.check(0, "x")
    with pytest.raises(ValueError):
        C.check(C.RL_ERR_BAD_ARG, "x")
    with pytest.raises(R.UnknownAttribute.__mro__[1]):  # RelabError base
        C.check(C.RL_ERR_OUTPUT_TOO_LARGE, "x")
    with pytest.raises(RuntimeError):
        C.check(C.RL_ERR_CUDA + 700, "x")


def test_column_descriptor_array():
    arr, n = C.columns_array([(16, 32, 8, C.RL_SIDE_LEFT), (None, 64, 8, C.RL_SIDE_KEY)])
    assert n == 2 and arr[0].width == 8 and arr[1].side == C.RL_SIDE_KEY and arr[1].src is None
    with pytest.raises(ValueError):
        C.columns_array([(0, 0, 8, 0)] * (C.RL_MAX_COLUMNS + 1))


def test_operators_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2602_21237_b200 import Int64, Relation, Schema, tensor_sort, to_tensor, SortSpec

    rel = Relation(Schema((("key", Int64()),)), (np.array([2, 1], np.int64),))
    with pytest.raises(RuntimeError, match="CUDA"):
        to_tensor(rel, "key")
    with pytest.raises(RuntimeError, match="CUDA"):
        tensor_sort(rel, SortSpec(("key",)))
