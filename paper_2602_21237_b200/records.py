"""Relation, schema, spec and metrics records used at the operator boundary.

These restate the reference's I/O types for the tensor path so the package
runs stand-alone on a GPU box where ``relab`` is not installed:

* ``Int64`` / ``Bytes``            relation.py:23-40
* ``Schema``                       relation.py:46-89
* ``Relation`` (immutable numpy)   relation.py:92-208
* ``join_output_schema``           relation.py:337-357
* ``Direction``/``SortSpec``/``MemoryBudget``/``JoinSpec``  specs.py:12-65
* ``SpillStats``                   spill.py:26-48

The operators in ``tensor_path`` only duck-type these (``.schema.attributes``,
``.columns``, ``type(rel)(schema, cols)``), so they accept and return the
reference's own classes unchanged when installed into ``relab``.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from enum import Enum
from typing import Iterable, Optional, Sequence, Union

import numpy as np

from .errors import UnknownAttribute

BLOCK_SIZE = 8192  # spill.py:21 — only used to express temp_mb
MIN_BUDGET_BYTES = 65536  # specs.py:9


@dataclass(frozen=True)
class Int64:
    """Signed 64-bit attribute; serialised as 8 little-endian bytes."""

    @property
    def width(self) -> int:
        return 8


@dataclass(frozen=True)
class Bytes:
    """Opaque fixed-width attribute of ``width`` bytes (width may be 0)."""

    width: int

    def __post_init__(self) -> None:
        if self.width < 0:
            raise ValueError(f"byte attribute width must be >= 0, got {self.width}")


ColumnType = Union[Int64, Bytes]


def is_int64(t) -> bool:
    """True for an Int64 attribute type, whichever package defined it."""
    return type(t).__name__ == "Int64"


@dataclass(frozen=True)
class Schema:
    """Ordered, uniquely named attributes."""

    attributes: tuple

    def __post_init__(self) -> None:
        attrs = tuple((str(name), t) for name, t in self.attributes)
        if not attrs:
            raise ValueError("schema needs at least one attribute")
        seen = set()
        for name, _ in attrs:
            if not name:
                raise ValueError("attribute names must be non-empty")
            if name in seen:
                raise ValueError(f"duplicate attribute names in {[n for n, _ in attrs]}")
            seen.add(name)
        object.__setattr__(self, "attributes", attrs)

    @property
    def names(self) -> tuple:
        return tuple(name for name, _ in self.attributes)

    def index(self, name: str) -> int:
        for i, (n, _) in enumerate(self.attributes):
            if n == name:
                return i
        raise UnknownAttribute(name)

    def type_of(self, name: str) -> ColumnType:
        return self.attributes[self.index(name)][1]

    @property
    def row_width(self) -> int:
        return sum(t.width for _, t in self.attributes)

    @property
    def offsets(self) -> tuple:
        out, pos = [], 0
        for _, t in self.attributes:
            out.append(pos)
            pos += t.width
        return tuple(out)


def _frozen_column(col, ctype) -> np.ndarray:
    if is_int64(ctype):
        arr = np.ascontiguousarray(col, dtype=np.int64)
        if arr.ndim != 1:
            raise ValueError("int64 columns must be 1-D")
    else:
        arr = np.ascontiguousarray(col, dtype=np.uint8)
        if arr.ndim != 2 or arr.shape[1] != ctype.width:
            raise ValueError(f"byte column must have shape (n, {ctype.width}), got {arr.shape}")
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class Relation:
    """A schema plus one read-only numpy column per attribute."""

    schema: Schema
    columns: tuple

    def __post_init__(self) -> None:
        if len(self.columns) != len(self.schema.attributes):
            raise ValueError("column count does not match schema")
        cols = tuple(_frozen_column(c, t) for c, (_, t) in zip(self.columns, self.schema.attributes))
        if len({len(c) for c in cols}) > 1:
            raise ValueError(f"columns have differing lengths: {sorted({len(c) for c in cols})}")
        object.__setattr__(self, "columns", cols)

    @property
    def row_count(self) -> int:
        return len(self.columns[0])

    def column(self, name: str) -> np.ndarray:
        return self.columns[self.schema.index(name)]

    def take(self, indices) -> "Relation":
        idx = np.asarray(indices, dtype=np.int64)
        return Relation(self.schema, tuple(c[idx] for c in self.columns))

    def serialize(self) -> np.ndarray:
        """Canonical (n, row_width) little-endian row bytes."""
        n = self.row_count
        out = np.empty((n, self.schema.row_width), dtype=np.uint8)
        for col, (_, t), off in zip(self.columns, self.schema.attributes, self.schema.offsets):
            if is_int64(t):
                out[:, off : off + 8] = col.astype("<i8", copy=False).view(np.uint8).reshape(n, 8)
            elif t.width:
                out[:, off : off + t.width] = col
        return out

    def row_tuples(self) -> list:
        parts = []
        for col, (_, t) in zip(self.columns, self.schema.attributes):
            if is_int64(t):
                parts.append(col.tolist())
            else:
                parts.append([bytes(r) for r in col] if t.width else [b""] * len(col))
        return list(zip(*parts))

    @classmethod
    def from_rows(cls, schema: Schema, rows: Iterable[tuple]) -> "Relation":
        rows = list(rows)
        cols = []
        for i, (_, t) in enumerate(schema.attributes):
            if is_int64(t):
                cols.append(np.array([r[i] for r in rows], dtype=np.int64))
            else:
                raw = b"".join(r[i] for r in rows)
                cols.append(np.frombuffer(raw, dtype=np.uint8).reshape(len(rows), t.width))
        return cls(schema, tuple(cols))

    @classmethod
    def empty(cls, schema: Schema) -> "Relation":
        return cls(
            schema,
            tuple(
                np.empty(0, np.int64) if is_int64(t) else np.empty((0, t.width), np.uint8)
                for _, t in schema.attributes
            ),
        )


def join_output_schema(left, right, key: str, schema_cls=None):
    """Left attributes, then right non-key attributes; a colliding right name
    is prefixed with ``right_`` until unique (relation.py:337-357)."""
    if not is_int64(left.type_of(key)):
        raise UnknownAttribute(f"join key {key!r} must be int64 in left schema")
    if not is_int64(right.type_of(key)):
        raise UnknownAttribute(f"join key {key!r} must be int64 in right schema")
    attrs = list(left.attributes)
    used = {name for name, _ in attrs}
    for name, t in right.attributes:
        if name == key:
            continue
        out = name
        while out in used:
            out = "right_" + out
        used.add(out)
        attrs.append((out, t))
    return (schema_cls or type(left))(tuple(attrs))


class Direction(Enum):
    ASC = "asc"
    DESC = "desc"


class BuildSide(Enum):
    LEFT = "left"
    RIGHT = "right"


@dataclass(frozen=True)
class MemoryBudget:
    """work_mem analogue; at least 64 KiB (specs.py:22-32)."""

    bytes: int

    def __post_init__(self) -> None:
        if self.bytes < MIN_BUDGET_BYTES:
            raise ValueError(f"budget must be >= {MIN_BUDGET_BYTES} bytes, got {self.bytes}")


@dataclass(frozen=True)
class JoinSpec:
    key: str
    build_side: Optional[BuildSide] = None


@dataclass(frozen=True)
class SortSpec:
    """Sort keys, most significant first, each with a direction (ASC default)."""

    keys: tuple
    directions: tuple = ()

    def __post_init__(self) -> None:
        keys = tuple(self.keys)
        if not keys:
            raise ValueError("sort needs at least one key")
        if len(set(keys)) != len(keys):
            raise ValueError(f"duplicate sort keys in {keys}")
        dirs = tuple(d if isinstance(d, Direction) else Direction(d) for d in self.directions)
        if not dirs:
            dirs = (Direction.ASC,) * len(keys)
        if len(dirs) != len(keys):
            raise ValueError("directions must match keys in length")
        object.__setattr__(self, "keys", keys)
        object.__setattr__(self, "directions", dirs)


def is_descending(direction) -> bool:
    """Direction test that accepts this package's or relab's enum (or a str)."""
    value = getattr(direction, "value", direction)
    return str(value).lower() == "desc"


@dataclass
class SpillStats:
    """Per-operator counters (spill.py:26-48). The GPU path never touches
    temp files, so every temp_* field stays 0; peak_* is device accounting."""

    temp_bytes_written: int = 0
    temp_blocks_written: int = 0
    temp_bytes_read: int = 0
    partition_passes: int = 0
    sort_runs: int = 0
    peak_mem_bytes: int = 0
    peak_build_bytes: int = 0

    @property
    def temp_mb(self) -> float:
        return self.temp_blocks_written * BLOCK_SIZE / 2**20

    def copy(self) -> "SpillStats":
        return replace(self)
