"""Drop-in tensor path: the reference operator API on B200 kernels.

Same names, signatures, return types and error behaviour as
/root/reference/pkg/src/relab/tensorpath.py:

    to_tensor(rel, key) -> TensorRelation                      (tensorpath.py:78)
    key_axis_align(left, right) -> AxisAlignment               (tensorpath.py:109)
    tensor_join(left, right, max_output_rows=2**31)
        -> (Relation, SpillStats)                              (tensorpath.py:131)
    tensor_sort(rel, spec) -> (Relation, SpillStats)           (tensorpath.py:232)

Inputs are numpy-backed Relations (this package's or relab's own); the key
column and the payload axes are copied to HBM once per ``to_tensor``, every
primitive runs as an sm_100a kernel (engine.py), and outputs come back as
fresh read-only numpy columns of the input's Relation class. A join
synchronises the host exactly once (to size its output). The index arrays of
TensorRelation / AxisAlignment stay on the device and are copied to numpy
only when a caller reads them.
"""

from __future__ import annotations

import ctypes
import sys
import warnings
import weakref
from collections import OrderedDict
from typing import Optional

import numpy as np
import torch

from . import _capi as C
from . import engine
from . import errors as _errors
from . import records as _records
from .records import is_descending, is_int64

MAX_OUTPUT_ROWS = 2**31  # tensorpath.py:22

# Record/exception classes the operators construct or raise. patch.install()
# rebinds them to relab's classes so a patched relab sees its own types.
TYPES = {
    "SpillStats": _records.SpillStats,
    "OutputTooLarge": _errors.OutputTooLarge,
    "UnknownAttribute": _errors.UnknownAttribute,
}

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 tensor path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


_STAGE_MIN_BYTES = 1 << 20
_stagers: dict = {}


def _stager(dev) -> int:
    """Per-device native staging pipeline (csrc/stager.cu): pinned ring of
    4 x 8 MiB, up to 8 copy threads, its own copy stream."""
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    h = _stagers.get(idx)
    if h is None:
        import os

        threads = max(1, min(8, (os.cpu_count() or 2) // 2))
        h = C.load().rl_stager_create(threads, 8 << 20, 4)
        if not h:
            raise RuntimeError("rl_stager_create failed (pinned host memory / CUDA stream)")
        _stagers[idx] = h
    return h


_REGISTER_MIN_BYTES = 4 << 20
# id(owner) -> (ptr, nbytes, finalizer): page-locked ranges of live numpy
# buffers, least recently used first; their total stays within _pin_budget()
_registered: "OrderedDict[int, tuple]" = OrderedDict()


def _pin_budget() -> int:
    """Bytes of caller memory the drop-in may keep page-locked at once:
    RL_PIN_BUDGET_BYTES, default a quarter of physical memory capped at
    16 GiB. Past it the least recently used registrations are released."""
    import os

    v = os.environ.get("RL_PIN_BUDGET_BYTES")
    if v:
        return max(0, int(v))
    try:
        phys = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError, AttributeError):
        phys = 16 << 30
    return min(16 << 30, phys // 4)


def pinned_bytes() -> int:
    """Caller memory currently page-locked by the drop-in (≤ _pin_budget())."""
    return sum(v[1] for v in _registered.values())


def _evict_pins(need: int, budget: int) -> None:
    """Release least recently used registrations until `need` more bytes fit."""
    while _registered and pinned_bytes() + need > budget:
        _key, (_ptr, _n, fin) = next(iter(_registered.items()))
        fin()  # drains the stager, unregisters, drops the entry


def _owner(arr: np.ndarray):
    while isinstance(arr.base, np.ndarray):
        arr = arr.base
    return arr


def _page_locked(arr: np.ndarray, dev) -> bool:
    """Page-lock a large input column's memory once, for as long as its
    numpy buffer lives, so every later upload of it is one direct DMA.

    Relations are immutable and the reference harness reuses its inputs
    across repetitions (bench.py:219-224), so this is the pinned-input fast
    path; anything that cannot be registered (foreign buffers, ranges that
    share pages with another registration) uses the staging pipeline."""
    lib = C.load()
    if lib.rl_host_is_pinned(ctypes.c_void_p(arr.ctypes.data)) and lib.rl_host_is_pinned(
            ctypes.c_void_p(arr.ctypes.data + arr.nbytes - 1)):
        return True  # already page-locked (e.g. a previous operator's pinned output)
    own = _owner(arr)
    if own.nbytes > 4 * arr.nbytes:  # a small view of a huge buffer: stage it instead
        return False
    ptr, nbytes = own.ctypes.data, own.nbytes
    key = id(own)
    hit = _registered.get(key)
    if hit is not None:
        _registered.move_to_end(key)
        p0, n0, _ = hit
        return p0 <= arr.ctypes.data and arr.ctypes.data + arr.nbytes <= p0 + n0
    budget = _pin_budget()
    if nbytes > budget:
        return False
    _evict_pins(nbytes, budget)
    if lib.rl_host_register(ctypes.c_void_p(ptr), nbytes) != C.RL_OK:
        return False
    stager = _stager(dev)

    def _release(ptr=ptr, key=key, stager=stager, lib=lib):
        lib.rl_stager_drain(stager)  # no DMA may still read the buffer
        lib.rl_host_unregister(ctypes.c_void_p(ptr))
        _registered.pop(key, None)

    try:
        fin = weakref.finalize(own, _release)
    except TypeError:  # owner not weak-referenceable: keep it registered only for this call
        lib.rl_host_unregister(ctypes.c_void_p(ptr))
        return False
    _registered[key] = (ptr, nbytes, fin)
    return True


class _Uploads:
    """Device destinations for host columns, allocated up front.

    All destinations are allocated, then one event is recorded on the
    current stream; every staged upload waits only for that event, so it
    cannot overtake earlier work on recycled allocator memory, while the
    kernels enqueued afterwards (the key sort) overlap the payload uploads.
    """

    def __init__(self, arrays, dev):
        self.host = [np.ascontiguousarray(a) for a in arrays]
        self.dev = []
        for a in self.host:
            if a.dtype not in (np.int64, np.uint8, np.int32):
                raise ValueError(f"unsupported column dtype {a.dtype}")
            dt = {np.dtype(np.int64): torch.int64, np.dtype(np.uint8): torch.uint8, np.dtype(np.int32): torch.int32}
            self.dev.append(torch.empty(a.shape, dtype=dt[a.dtype], device=dev))
        self.ready = torch.cuda.Event()
        self.ready.record()
        self.done = [False] * len(self.host)

    def get(self, j: int) -> torch.Tensor:
        """Device copy of column j, uploading it now if it has not been."""
        if not self.done[j]:
            arr, out = self.host[j], self.dev[j]
            if arr.nbytes >= _REGISTER_MIN_BYTES and _page_locked(arr, out.device):
                C.check(C.load().rl_stager_h2d_pinned(_stager(out.device), ctypes.c_void_p(out.data_ptr()),
                                                      ctypes.c_void_p(arr.ctypes.data), arr.nbytes,
                                                      engine.stream_handle(), ctypes.c_void_p(self.ready.cuda_event)),
                        "rl_stager_h2d_pinned")
            elif arr.nbytes >= _STAGE_MIN_BYTES:
                C.check(C.load().rl_stager_h2d(_stager(out.device), ctypes.c_void_p(out.data_ptr()),
                                               ctypes.c_void_p(arr.ctypes.data), arr.nbytes,
                                               engine.stream_handle(), ctypes.c_void_p(self.ready.cuda_event)),
                        "rl_stager_h2d")
            elif arr.nbytes:
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", UserWarning)
                    out.copy_(torch.from_numpy(arr))
            self.done[j] = True
        return self.dev[j]


def _h2d(arr: np.ndarray, dev) -> torch.Tensor:
    """One host column → HBM (int64 [n], int32 [n] or uint8 [n, w])."""
    return _Uploads([arr], dev).get(0)


def _to_numpy_i64(dev_u32_or_i64: torch.Tensor, n: int) -> np.ndarray:
    if n == 0:
        out = np.empty(0, dtype=np.int64)
    elif dev_u32_or_i64.dtype == torch.int64:
        out = dev_u32_or_i64[:n].cpu().numpy()
    else:
        out = engine.widen(dev_u32_or_i64, n).cpu().numpy()
    out.setflags(write=False)
    return out


class TensorRelation:
    """Attribute axes plus the sorted sparse key axis (tensorpath.py:25-59).

    ``key_values`` (strictly increasing distinct keys), ``offsets`` (CSR run
    starts, D+1 entries) and ``positions`` (rows grouped by key, each group in
    row order) are int64 numpy arrays like the reference's; here they live in
    HBM and are copied out only when read. ``axes`` are the input columns
    unchanged, so ``to_relation`` is the identity.
    """

    __slots__ = ("schema", "axes", "key", "_index", "_dev_axes", "_d", "_cache")

    def __init__(self, schema, axes, key, key_values=None, offsets=None, positions=None, *, _index=None,
                 _dev_axes=None):
        self.schema = schema
        self.axes = tuple(axes)
        self.key = key
        self._index = _index
        self._dev_axes = _dev_axes
        self._d = None
        self._cache = {}
        if _index is None:
            # constructed from host arrays, as the reference dataclass is
            kv = np.asarray(key_values, dtype=np.int64)
            off = np.asarray(offsets, dtype=np.int64)
            pos = np.asarray(positions, dtype=np.int64)
            if len(off) != len(kv) + 1:
                raise ValueError("offsets must have one more entry than key_values")
            if len(kv) and not (np.diff(kv) > 0).all():
                raise ValueError("key_values must be strictly increasing")
            if (len(off) and off[0] != 0) or (np.diff(off) < 0).any():
                raise ValueError("offsets must start at 0 and be non-decreasing")
            if off[-1] != len(pos):
                raise ValueError("final offset must equal row count")
            self._cache = {"key_values": kv, "offsets": off, "positions": pos}
            self._d = len(kv)

    def __setattr__(self, name, value):
        if name in ("schema", "axes", "key") and hasattr(self, name):
            raise AttributeError(f"TensorRelation.{name} is read-only")
        object.__setattr__(self, name, value)

    # -- device side ---------------------------------------------------
    def device_index(self) -> engine.KeyIndex:
        if self._index is None:  # host-constructed: upload once
            dev = _device()
            n = len(self._cache["positions"])
            kv = self._cache["key_values"]
            d = len(kv)
            idx = engine.KeyIndex(
                n,
                _h2d(kv if d else np.zeros(1, np.int64), dev),
                _h2d(self._cache["offsets"].astype(np.uint32).view(np.int32), dev),
                _h2d(self._cache["positions"].astype(np.uint32).view(np.int32), dev),
                torch.tensor([d], dtype=torch.int64, device=dev),
            )
            object.__setattr__(self, "_index", idx)
        return self._index

    def device_axes(self) -> tuple:
        if self._dev_axes is None:
            dev = _device()
            object.__setattr__(self, "_dev_axes", tuple(_h2d(a, dev) for a in self.axes))
        return self._dev_axes

    def distinct_count(self) -> int:
        if self._d is None:
            object.__setattr__(self, "_d", int(engine.fetch_scalars(self._index.d)[0]))
        return self._d

    # -- reference fields ----------------------------------------------
    @property
    def key_values(self) -> np.ndarray:
        if "key_values" not in self._cache:
            self._cache["key_values"] = _to_numpy_i64(self._index.key_values, self.distinct_count())
        return self._cache["key_values"]

    @property
    def offsets(self) -> np.ndarray:
        if "offsets" not in self._cache:
            self._cache["offsets"] = _to_numpy_i64(self._index.offsets, self.distinct_count() + 1)
        return self._cache["offsets"]

    @property
    def positions(self) -> np.ndarray:
        if "positions" not in self._cache:
            self._cache["positions"] = _to_numpy_i64(self._index.positions, self._index.n)
        return self._cache["positions"]

    @property
    def row_count(self) -> int:
        return self._index.n if self._index is not None else len(self._cache["positions"])

    def to_relation(self):
        return _relation_class_of(self)(self.schema, self.axes)

    def __repr__(self) -> str:
        return f"TensorRelation(key={self.key!r}, rows={self.row_count}, device=True)"


def _relation_class_of(t) -> type:
    """The Relation class that goes with t's schema: the module defining the
    Schema class defines Relation too (relab.relation or records)."""
    mod = sys.modules.get(type(t.schema).__module__)
    return getattr(mod, "Relation", _records.Relation)


def to_tensor(rel, key: str) -> TensorRelation:
    """Index a relation on its int64 join key with a stable (key, row) radix
    sort on the B200 (tensorpath.py:78-93). All axes are staged in HBM."""
    if not is_int64(rel.schema.type_of(key)):
        raise TYPES["UnknownAttribute"](f"key attribute {key!r} must be int64")
    dev = _device()
    key_idx = rel.schema.index(key)
    up = _Uploads(rel.columns, dev)
    index = engine.index_keys(up.get(key_idx))  # queued behind the key upload only
    dev_axes = tuple(up.get(j) for j in range(len(rel.columns)))  # overlap the sort
    return TensorRelation(rel.schema, rel.columns, key, _index=index, _dev_axes=dev_axes)


class AxisAlignment:
    """Intersection of two key axes with both sides' grouped positions
    (tensorpath.py:96-106); fields are int64 numpy arrays read lazily."""

    def __init__(self, left: TensorRelation, right: TensorRelation, dev: engine.Alignment):
        self._left, self._right, self._dev = left, right, dev
        self._m = None
        self._cache = {}

    @property
    def device(self) -> engine.Alignment:
        return self._dev

    def _count(self) -> int:
        if self._m is None:
            self._m = int(engine.fetch_scalars(self._dev.m_total[:1])[0])
        return self._m

    def _field(self, name, tensor):
        if name not in self._cache:
            self._cache[name] = _to_numpy_i64(tensor, self._count())
        return self._cache[name]

    @property
    def matched_keys(self):
        return self._field("matched_keys", self._dev.matched_keys)

    @property
    def left_starts(self):
        return self._field("left_starts", self._dev.left_starts)

    @property
    def left_counts(self):
        return self._field("left_counts", self._dev.left_counts)

    @property
    def right_starts(self):
        return self._field("right_starts", self._dev.right_starts)

    @property
    def right_counts(self):
        return self._field("right_counts", self._dev.right_counts)

    @property
    def left_positions(self):
        return self._left.positions

    @property
    def right_positions(self):
        return self._right.positions


def key_axis_align(left: TensorRelation, right: TensorRelation) -> AxisAlignment:
    """Match the two sorted distinct-key axes on the device (tensorpath.py:109-128)."""
    left, right = _as_device_tensor(left), _as_device_tensor(right)
    return AxisAlignment(left, right, engine.align(left.device_index(), right.device_index()))


def _as_device_tensor(t) -> TensorRelation:
    """Accept a reference TensorRelation (numpy fields) as well as ours."""
    if isinstance(t, TensorRelation):
        return t
    return TensorRelation(t.schema, t.axes, t.key, t.key_values, t.offsets, t.positions)


_D2H_STREAMS: dict = {}


def _d2h_stream(dev) -> torch.cuda.Stream:
    key = torch.device(dev).index
    if key not in _D2H_STREAMS:
        _D2H_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _D2H_STREAMS[key]


def _host_out_on(dev_t: torch.Tensor, stream: torch.cuda.Stream) -> torch.Tensor:
    """D2H of dev_t on `stream` once the current stream's work so far is done."""
    host = torch.empty(dev_t.shape, dtype=dev_t.dtype, pin_memory=True)
    ready = torch.cuda.Event()
    ready.record()
    stream.wait_event(ready)
    with torch.cuda.stream(stream):
        host.copy_(dev_t, non_blocking=True)
    dev_t.record_stream(stream)
    return host


def _host_out(dev_t: torch.Tensor) -> torch.Tensor:
    host = torch.empty(dev_t.shape, dtype=dev_t.dtype, pin_memory=True)
    host.copy_(dev_t, non_blocking=True)
    return host


def tensor_join(left: TensorRelation, right: TensorRelation, max_output_rows: int = MAX_OUTPUT_ROWS):
    """Equi-join by key-axis alignment on the B200; never spills.

    Output rows are ordered (key, left row, right row), byte-identical to the
    reference (tensorpath.py:157-172). Raises OutputTooLarge before any
    output allocation when the pair count exceeds ``max_output_rows``.
    """
    if left.key != right.key:
        raise TYPES["UnknownAttribute"](f"inputs indexed on different keys: {left.key!r} vs {right.key!r}")
    left, right = _as_device_tensor(left), _as_device_tensor(right)
    li, ri = left.device_index(), right.device_index()
    al = engine.align(li, ri)
    rel_cls = _relation_class_of(left)
    out_schema = _records.join_output_schema(left.schema, right.schema, left.key, schema_cls=type(left.schema))
    d_l, d_r, m, total = engine.fetch_scalars(li.d, ri.d, al.m_total)
    if total > max_output_rows:
        raise TYPES["OutputTooLarge"](f"join would produce {total} rows (cap {max_output_rows})")
    if total == 0:
        return rel_cls.empty(out_schema), TYPES["SpillStats"]()

    from .pipeline import join_out_columns

    cols = join_out_columns(left.device_axes(), left.schema.index(left.key), right.device_axes(),
                            right.schema.index(right.key), total)
    engine.expand(al, m, li, ri, 0, total, cols)
    hosts = [_host_out(c.dst) for c in cols]
    torch.cuda.current_stream().synchronize()
    out = rel_cls(out_schema, tuple(h.numpy() for h in hosts))

    out_bytes = sum(c.dst.numel() * c.dst.element_size() for c in cols)
    stats = TYPES["SpillStats"](peak_mem_bytes=join_peak_mem_bytes(li.n, d_l, ri.n, d_r, total, out_bytes),
                                peak_build_bytes=0)
    return out, stats


def join_peak_mem_bytes(n_left: int, d_left: int, n_right: int, d_right: int, total: int, out_bytes: int) -> int:
    """SpillStats.peak_mem_bytes of a join, the reference's closed form
    (tensorpath.py:188-202): the int64 index arrays of both sides, the
    expansion temporaries (4 index-dtype arrays + 4 int64 arrays per pair;
    int32 indices when total <= 2^31 - 1, tensorpath.py:159) and the output
    columns — the same deterministic number the reference records."""
    index_bytes = 8 * (n_left + n_right) + 8 * (d_left + d_right) + 8 * (d_left + 1 + d_right + 1)
    idx_size = 4 if total <= 2**31 - 1 else 8
    return index_bytes + total * (4 * idx_size + 4 * 8) + out_bytes


def sort_peak_mem_bytes(n: int, out_bytes: int) -> int:
    """SpillStats.peak_mem_bytes of a sort, the reference's closed form
    (tensorpath.py:248-251): two int64 permutations + the output columns."""
    return 2 * 8 * n + out_bytes


def _out_column(src: torch.Tensor, ctype, rows: int, dev, side: int) -> engine.OutColumn:
    if is_int64(ctype):
        return engine.OutColumn(src, torch.empty(rows, dtype=torch.int64, device=dev), 8, side)
    w = ctype.width
    return engine.OutColumn(src, torch.empty((rows, w), dtype=torch.uint8, device=dev), w, side)


def tensor_sort(rel, spec):
    """Multi-key stable sort on the B200 (tensorpath.py:232-252): LSD over the
    key axes with per-word radix passes, then one gather of every column.
    Tie order and DESC semantics equal the comparator oracle's."""
    for k in spec.keys:
        rel.schema.index(k)  # UnknownAttribute for a missing key
    n = rel.row_count
    rel_cls = type(rel)
    if n == 0:
        return rel_cls(rel.schema, rel.columns), TYPES["SpillStats"](peak_mem_bytes=0, peak_build_bytes=0)
    dev = _device()
    up = _Uploads(rel.columns, dev)
    axes = [engine.SortAxis(up.get(rel.schema.index(k)), is_descending(d)) for k, d in zip(spec.keys, spec.directions)]
    single_int = len(axes) == 1 and axes[0].is_int64
    key_j = rel.schema.index(spec.keys[0])
    sorted_key = torch.empty(n, dtype=torch.int64, device=dev) if single_int else None
    perm = engine.sort_permutation(axes, n, dev, sorted_keys_out=sorted_key)
    # PCIe is full duplex: the sorted key column goes down on its own stream
    # while the payload columns are still coming up for the gather
    down = _d2h_stream(dev)
    hosts = [None] * len(rel.columns)
    if single_int:
        hosts[key_j] = _host_out_on(sorted_key, down)
    outs, gathers, idx = [], [], []
    for j, (_, t) in enumerate(rel.schema.attributes):
        if single_int and j == key_j:
            outs.append(sorted_key)
            continue
        col = _out_column(up.get(j), t, n, dev, C.RL_SIDE_LEFT)  # uploads overlap the sort
        gathers.append(col)
        outs.append(col.dst)
        idx.append(j)
    engine.gather_rows(perm, gathers)
    for j, col in zip(idx, gathers):
        hosts[j] = _host_out_on(col.dst, down)
    down.synchronize()
    out = rel_cls(rel.schema, tuple(h.numpy() for h in hosts))
    stats = TYPES["SpillStats"](peak_mem_bytes=sort_peak_mem_bytes(n, sum(o.numel() * o.element_size() for o in outs)),
                                peak_build_bytes=0)
    return out, stats


def multiset_digest(rel) -> int:
    """relation.py:319-330 on the device: XOR of the per-row 128-bit hashes of
    the canonical serialisation, computed straight from the columns (no
    serialised copy). Returns the digest as an int (``ResultDigest.value``)."""
    if rel.row_count == 0:
        return 0
    dev = _device()
    up = _Uploads(rel.columns, dev)
    return engine.multiset_digest([up.get(j) for j in range(len(rel.columns))])
