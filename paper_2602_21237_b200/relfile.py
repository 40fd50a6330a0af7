"""RELCOL01 relation files straight to / from HBM and page-locked memory.

The reference stores relations as ``b"RELCOL01"``, a 4-byte little-endian
header length, a JSON header ``{"attrs": [[name, "int64" | ["bytes", w]], ...],
"rows": n}`` and then one section per column in canonical serialisation
(int64 little-endian, Bytes(w) row-major) — relation.py:364-419
(``write_relation`` / ``read_relation``). Files written here are
byte-identical to the reference's and files it writes are read here.

SURVEY.md §8(f) row 4: inputs shared across ranks and runs (1e8-1e9 rows)
should not round-trip through numpy. ``read_device`` reads every column
section with the native stager (csrc/stager.cu: parallel ``pread`` into a
pinned ring, the copy engine DMAs the previous chunk to HBM meanwhile);
``write_device`` goes the other way through the same ring; ``read_pinned``
reads into page-locked numpy columns, so the drop-in operators upload them
with one direct DMA each. ``read_device(path, rows=(a, b))`` reads the row
range [a, b) of every column — one rank's shard of a shared file.
"""

from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path
from typing import List, Optional, Tuple, Union

import numpy as np
import torch

from . import _capi as C
from . import engine
from . import records as R

MAGIC = b"RELCOL01"
PathLike = Union[str, Path]


def _type_from_json(obj):
    if obj == "int64":
        return R.Int64()
    if isinstance(obj, list) and len(obj) == 2 and obj[0] == "bytes":
        return R.Bytes(int(obj[1]))
    raise ValueError(f"unknown column type {obj!r}")


def _type_to_json(t):
    return "int64" if R.is_int64(t) else ["bytes", t.width]


def _width(t) -> int:
    return 8 if R.is_int64(t) else int(t.width)


def header_bytes(schema, rows: int) -> bytes:
    """Magic + length + JSON header exactly as relation.py:379-392 writes them."""
    header = json.dumps({"attrs": [[n, _type_to_json(t)] for n, t in schema.attributes], "rows": int(rows)}).encode()
    return MAGIC + len(header).to_bytes(4, "little") + header


def read_header(path: PathLike, schema_cls=None):
    """(schema, rows, [(file offset, bytes per row) per column]) — the checks of
    relation.py:398-419 (bad magic, truncated sections) raise ValueError."""
    path = Path(path)
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ValueError(f"{path}: not a relation file")
        hlen = int.from_bytes(f.read(4), "little")
        header = json.loads(f.read(hlen))
    n = int(header["rows"])
    schema = (schema_cls or R.Schema)(tuple((name, _type_from_json(t)) for name, t in header["attrs"]))
    off, sections = 12 + hlen, []
    for _, t in schema.attributes:
        sections.append((off, _width(t)))
        off += n * _width(t)
    if path.stat().st_size < off:
        raise ValueError(f"{path}: truncated column section")
    return schema, n, sections


def _stager(dev) -> int:
    from .tensor_path import _stager as get

    return get(torch.device(dev))


def read_device(path: PathLike, device=None, rows: Optional[Tuple[int, int]] = None):
    """A relation file → pipeline.DeviceRelation (columns in HBM), optionally
    only the row range ``rows = (a, b)``."""
    from .pipeline import DeviceRelation
    from .tensor_path import _device

    dev = torch.device(device) if device is not None else _device()
    schema, n, sections = read_header(path)
    a, b = rows if rows is not None else (0, n)
    if not 0 <= a <= b <= n:
        raise ValueError(f"row range {rows} outside [0, {n}]")
    m = b - a
    lib = C.load()
    stager = _stager(dev)
    ready = torch.cuda.Event()
    cols: List[torch.Tensor] = []
    for (_, t) in schema.attributes:
        cols.append(torch.empty(m, dtype=torch.int64, device=dev) if R.is_int64(t)
                    else torch.empty((m, t.width), dtype=torch.uint8, device=dev))
    ready.record()
    fd = os.open(str(path), os.O_RDONLY)
    try:
        for col, (off, w) in zip(cols, sections):
            if m and w:
                C.check(lib.rl_stager_file_h2d(stager, ctypes.c_void_p(col.data_ptr()), fd, off + a * w, m * w,
                                               engine.stream_handle(), ctypes.c_void_p(ready.cuda_event)),
                        "rl_stager_file_h2d")
    finally:
        os.close(fd)  # every pread has returned; only DMAs from the pinned ring may still be in flight
    return DeviceRelation(schema, cols)


def write_device(rel, path: PathLike) -> None:
    """pipeline.DeviceRelation → relation file, byte-identical to
    relation.py:379-392 (write_relation) for the same relation."""
    lib = C.load()
    n = rel.row_count
    dev = rel.columns[0].device if rel.columns else torch.device("cuda", torch.cuda.current_device())
    stager = _stager(dev)
    head = header_bytes(rel.schema, n)
    fd = os.open(str(path), os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        os.write(fd, head)
        off = len(head)
        for col, (_, t) in zip(rel.columns, rel.schema.attributes):
            w = _width(t)
            if n and w:
                col = col.contiguous()
                C.check(lib.rl_stager_file_d2h(stager, ctypes.c_void_p(col.data_ptr()), fd, off, n * w,
                                               engine.stream_handle()), "rl_stager_file_d2h")
            off += n * w
        os.ftruncate(fd, off)
    finally:
        os.close(fd)


def read_pinned(path: PathLike, relation_cls=None):
    """A relation file → Relation whose numpy columns live in page-locked
    memory (parallel pread straight into them)."""
    schema, n, sections = read_header(path)
    lib = C.load()
    stager = _stager(torch.device("cuda", torch.cuda.current_device()))
    cols = []
    fd = os.open(str(path), os.O_RDONLY)
    try:
        for (off, w), (_, t) in zip(sections, schema.attributes):
            buf = (torch.empty(n, dtype=torch.int64, pin_memory=True) if R.is_int64(t)
                   else torch.empty((n, t.width), dtype=torch.uint8, pin_memory=True))
            if n and w:
                C.check(lib.rl_stager_file_read(stager, ctypes.c_void_p(buf.data_ptr()), fd, off, n * w),
                        "rl_stager_file_read")
            cols.append(buf.numpy())
    finally:
        os.close(fd)
    cls = relation_cls or R.Relation
    return cls(schema, tuple(cols))
