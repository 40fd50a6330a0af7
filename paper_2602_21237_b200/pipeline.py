"""Device-resident relations and operator pipelines.

The drop-in operators (tensor_path) take and return numpy Relations, so a
join followed by an ORDER BY pays a D2H and an H2D round trip in between.
Here the relation stays in HBM from the first upload to the final
download: ``DeviceRelation`` holds the schema and one CUDA tensor per
column, and ``join`` / ``order_by`` run the same sm_100a kernels as the
drop-in (identical results, byte for byte).

``join_stream`` covers joins too large to materialise (BASELINE cfg3:
2.29e12 pairs at 10M x 10M Zipf): the sizing pass gives the exact count and
the expansion runs chunk by chunk over the output range.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterator, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _capi as C
from . import engine
from . import records as R
from .errors import OutputTooLarge
from .records import is_descending, is_int64


@dataclass
class DeviceRelation:
    """A relation whose columns live in HBM: int64 [n] or uint8 [n, w]."""

    schema: object
    columns: List[torch.Tensor]

    @property
    def row_count(self) -> int:
        return int(self.columns[0].shape[0])

    def column(self, name: str) -> torch.Tensor:
        return self.columns[self.schema.index(name)]

    @classmethod
    def from_host(cls, rel, device=None) -> "DeviceRelation":
        from .tensor_path import _device, _Uploads

        up = _Uploads(rel.columns, device or _device())
        return cls(rel.schema, [up.get(j) for j in range(len(rel.columns))])

    def to_host(self, relation_cls=None):
        """One pinned D2H per column, one sync; read-only numpy columns."""
        hosts = []
        for c in self.columns:
            h = torch.empty(c.shape, dtype=c.dtype, pin_memory=True)
            h.copy_(c, non_blocking=True)
            hosts.append(h)
        torch.cuda.current_stream().synchronize()
        cls = relation_cls
        if cls is None:
            import sys

            cls = getattr(sys.modules.get(type(self.schema).__module__), "Relation", R.Relation)
        return cls(self.schema, tuple(h.numpy() for h in hosts))

    @classmethod
    def from_file(cls, path, device=None, rows=None) -> "DeviceRelation":
        """A RELCOL01 relation file (relation.py:364-419) straight into HBM,
        optionally only the row range ``rows = (a, b)`` (relfile.read_device)."""
        from .relfile import read_device

        return read_device(path, device, rows)

    def to_file(self, path) -> None:
        """Write a RELCOL01 file byte-identical to relation.write_relation's."""
        from .relfile import write_device

        write_device(self, path)

    def digest(self) -> int:
        """relation.py:319-330 multiset digest, computed on the device."""
        return engine.multiset_digest(self.columns) if self.row_count else 0


def _empty_like(col: torch.Tensor, rows: int) -> torch.Tensor:
    return torch.empty((rows,) + tuple(col.shape[1:]), dtype=col.dtype, device=col.device)


def _width(col: torch.Tensor) -> int:
    return col.element_size() * (col.shape[1] if col.dim() > 1 else 1)


JoinPlan = engine.JoinPlanDev


def plan_join(left_keys: torch.Tensor, right_keys: torch.Tensor, left_carry=(), right_carry=()):
    """Everything a join needs before its output size is known, on the
    device: the bucket join (csrc/bucket_join.cu) when the keys allow it
    (carrying the given payload columns with the rows), else to_tensor x2 +
    key_axis_align + sizing in one C call over one workspace
    (rl_join_plan_build). One host sync (the totals)."""
    return engine.plan_join(left_keys, right_keys, left_carry, right_carry)


def join(left: DeviceRelation, right: DeviceRelation, key: str,
         max_output_rows: int = 2**31) -> DeviceRelation:
    """tensor_join on device relations (tensorpath.py:131-203): output rows in
    (key, left row, right row) order, columns = left attributes then right
    non-key attributes (join_output_schema)."""
    out_schema = R.join_output_schema(left.schema, right.schema, key, schema_cls=type(left.schema))
    lk, rk = left.schema.index(key), right.schema.index(key)
    plan = plan_join(left.columns[lk], right.columns[rk],
                     [c for j, c in enumerate(left.columns) if j != lk],
                     [c for j, c in enumerate(right.columns) if j != rk])
    if plan.total > max_output_rows:
        raise OutputTooLarge(f"join would produce {plan.total} rows (cap {max_output_rows})")
    cols = join_out_columns(left.columns, lk, right.columns, rk, plan.total)
    if plan.total:
        plan.expand(0, plan.total, cols)
    return DeviceRelation(out_schema, [c.dst for c in cols])


def join_out_columns(left_cols, left_key: int, right_cols, right_key: int, rows: int) -> List[engine.OutColumn]:
    """Output column descriptors of an equi-join (tensorpath.py:174-185): every
    left column (the key column is the matched key), then the right non-key
    columns."""
    cols = []
    for j, c in enumerate(left_cols):
        if j == left_key:
            cols.append(engine.OutColumn(None, _empty_like(c, rows), 8, C.RL_SIDE_KEY))
        else:
            cols.append(engine.OutColumn(c, _empty_like(c, rows), _width(c), C.RL_SIDE_LEFT))
    for j, c in enumerate(right_cols):
        if j != right_key:
            cols.append(engine.OutColumn(c, _empty_like(c, rows), _width(c), C.RL_SIDE_RIGHT))
    return cols


def order_by(rel: DeviceRelation, spec) -> Tuple[DeviceRelation, torch.Tensor]:
    """tensor_sort on a device relation (tensorpath.py:232-252). Returns the
    sorted relation and the permutation (uint32 bits in an int32 tensor)."""
    for k in spec.keys:
        rel.schema.index(k)
    n = rel.row_count
    dev = rel.columns[0].device
    axes = [engine.SortAxis(rel.column(k), is_descending(d)) for k, d in zip(spec.keys, spec.directions)]
    single_int = len(axes) == 1 and axes[0].is_int64
    key_j = rel.schema.index(spec.keys[0])
    sorted_key = torch.empty(n, dtype=torch.int64, device=dev) if single_int else None
    outs, gathers = [], []
    for j, c in enumerate(rel.columns):
        if single_int and j == key_j:
            outs.append(sorted_key)
            continue
        g = engine.OutColumn(c, _empty_like(c, n), _width(c), C.RL_SIDE_LEFT)
        gathers.append(g)
        outs.append(g.dst)
    import os

    if (os.environ.get("RL_SORT_CARRY", "") not in ("", "0") and single_int and n >= engine.CARRY_MIN_ROWS
            and engine.carry_fits(gathers) and engine.packable_keys(axes[0].data)):
        # opt-in: the other columns ride with the rows through the sort. Measured at
        # 1e8 (cfg5's ORDER BY, 16 carried bytes): 5.5 ms vs 5.3 ms sort + gather —
        # the carrying passes move 3x the bytes at 3-3.7 TB/s, the gather's 2
        # random reads a row cost about the same
        perm = engine.sort_carry(axes[0].data, axes[0].descending, sorted_key, gathers)
        return DeviceRelation(rel.schema, outs), perm
    perm = engine.sort_permutation(axes, n, dev, sorted_keys_out=sorted_key)
    if n:
        engine.gather_rows(perm, gathers)
    return DeviceRelation(rel.schema, outs), perm


def join_then_order_by(left: DeviceRelation, right: DeviceRelation, key: str, spec,
                       max_output_rows: int = 2**31) -> DeviceRelation:
    """BASELINE cfg5's pipeline without leaving HBM: equi-join, then ORDER BY.

    Fused layout (cfg5's shape: ORDER BY one int64 output column, the other
    output columns exactly two 8-byte columns, the bucket join's plan): the
    join writes the sort column as usual and the other two row-interleaved
    into one [rows, 16] buffer; the ORDER BY then takes each row of it with
    ONE random 16-byte load (rl_gather_rows_split16) instead of two 8-byte
    loads from two arrays — random gathers over a large output are bound by
    the access rate (scripts/microbench/gather_flavors.cu). The result equals
    join() then order_by() column for column (same permutation, same bytes).
    RL_NO_FUSED_ORDER_BY=1 runs the two steps as written."""
    import os

    out_schema = R.join_output_schema(left.schema, right.schema, key, schema_cls=type(left.schema))
    lk, rk = left.schema.index(key), right.schema.index(key)
    plan = plan_join(left.columns[lk], right.columns[rk],
                     [c for j, c in enumerate(left.columns) if j != lk],
                     [c for j, c in enumerate(right.columns) if j != rk])
    if plan.total > max_output_rows:
        raise OutputTooLarge(f"join would produce {plan.total} rows (cap {max_output_rows})")
    cols = join_out_columns(left.columns, lk, right.columns, rk, 0)  # (descriptors; outputs allocated below)
    for k in spec.keys:
        out_schema.index(k)
    fusable = (os.environ.get("RL_NO_FUSED_ORDER_BY", "") != "1" and getattr(plan, "kind", "") == "bucket"
               and plan.total > 0 and len(spec.keys) == 1 and len(cols) == 3)
    if fusable:
        j = out_schema.index(spec.keys[0])
        proto = [c.dst for c in cols]  # empty outputs of the right dtype / shape
        others = [i for i in range(3) if i != j]
        fusable = (proto[j].dtype == torch.int64 and proto[j].dim() == 1
                   and all(_width(proto[i]) == 8 for i in others))
    if not fusable:
        cols = join_out_columns(left.columns, lk, right.columns, rk, plan.total)
        if plan.total:
            plan.expand(0, plan.total, cols)
        joined = DeviceRelation(out_schema, [c.dst for c in cols])
        return order_by(joined, spec)[0]
    n = plan.total
    dev = proto[j].device
    sort_src = torch.empty(n, dtype=torch.int64, device=dev)
    inter = torch.empty((n, 16), dtype=torch.uint8, device=dev)
    halves = (inter[:, :8], inter[:, 8:])
    emit_cols, strides = [], []
    for i, c in enumerate(cols):
        if i == j:
            emit_cols.append(engine.OutColumn(c.src, sort_src, 8, c.side))
            strides.append(0)
        else:
            emit_cols.append(engine.OutColumn(c.src, halves[others.index(i)], 8, c.side))
            strides.append(16)
    plan.expand(0, n, emit_cols, dst_strides=strides)
    del plan
    sorted_key = torch.empty(n, dtype=torch.int64, device=dev)
    axis = engine.SortAxis(sort_src, is_descending(spec.directions[0]))
    perm = engine.sort_permutation([axis], n, dev, sorted_keys_out=sorted_key)
    del sort_src
    outs = [None, None, None]
    outs[j] = sorted_key
    for k, i in enumerate(others):
        outs[i] = _empty_like(proto[i], n)
    engine.gather_split16(perm, inter, outs[others[0]], outs[others[1]])
    return DeviceRelation(out_schema, outs)


def join_stream(plan: JoinPlan, chunk_pairs: int = 1 << 31, begin: int = 0,
                end: Optional[int] = None, out: Optional[Tuple[torch.Tensor, torch.Tensor]] = None
                ) -> Iterator[Tuple[int, torch.Tensor, torch.Tensor]]:
    """Materialise the (left row, right row) pairs of [begin, end) chunk by
    chunk (reference order), yielding (chunk start, left rows, right rows);
    the two uint32 buffers (``out``, or allocated here) are reused between
    chunks."""
    end = plan.total if end is None else min(end, plan.total)
    if end <= begin:
        return
    dev = plan.ws.device
    cap = min(chunk_pairs, end - begin)
    if out is not None and min(out[0].numel(), out[1].numel()) >= cap:
        lr, rr = out
    else:
        lr = torch.empty(cap, dtype=torch.int32, device=dev)
        rr = torch.empty(cap, dtype=torch.int32, device=dev)
    for a in range(begin, end, chunk_pairs):
        b = min(a + chunk_pairs, end)
        plan.expand(a, b, (), lr[: b - a], rr[: b - a])
        yield a, lr[: b - a], rr[: b - a]


def pair_checksum(plan: JoinPlan, begin: int = 0, end: Optional[int] = None) -> int:
    """Σ fmix64((left row << 32) | right row) mod 2^64 over pairs [begin, end)
    without materialising them (order-independent; the oracle's
    pair_checksum restricted to the same range agrees)."""
    end = plan.total if end is None else min(end, plan.total)
    acc = torch.zeros(1, dtype=torch.int64, device=plan.ws.device)
    if end > begin:
        plan.pair_checksum(begin, end, acc)
    return int(engine.fetch_scalars(acc)[0]) & (2**64 - 1)
