"""Device-resident execution of the tensor path on one B200.

Every function here takes and returns CUDA tensors and launches the sm_100a
kernels of librelab_b200.so on the current torch stream; nothing falls back to
the CPU. The numpy-facing drop-in (``tensor_path``) is a thin layer of H2D/D2H
copies around these calls, and the benchmark's device-resident numbers call
them directly with inputs already in HBM.

Kernel map:  index_keys = K1+K2 (radix sort) + K3 (run
bounds); align = K4+K5; expand = K6+K7 (fused); sort_permutation = K1+K2 per
key word; gather_rows = K7; hash_partition = K8.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import _capi as C

_U32 = torch.int32  # torch has no general uint32 tensor ops; bits are reinterpreted as uint32


def _require_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (the B200 path has no CPU fallback)")


def stream_handle(stream: Optional[torch.cuda.Stream] = None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def aligned16(t: torch.Tensor) -> torch.Tensor:
    """The sort streams int64 keys / row ids with 16-byte TMA bulk copies:
    give it a contiguous, 16-byte aligned view (copy only if needed)."""
    t = t.contiguous()
    return t if t.data_ptr() % 16 == 0 else t.clone()


def workspace(nbytes: int, device) -> torch.Tensor:
    """Scratch from torch's stream-ordered caching allocator (512 B aligned)."""
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


@dataclass
class KeyIndex:
    """The sparse key axis of one relation, on the device (to_tensor)."""

    n: int
    key_values: torch.Tensor  # int64, capacity max(n, 1); first D valid
    offsets: torch.Tensor  # uint32 bits, capacity n + 1; first D + 1 valid
    positions: torch.Tensor  # uint32 bits, n
    d: torch.Tensor  # int64 [1]: D (device scalar)

    def nbytes(self, d: int) -> int:
        return 4 * self.n + 8 * d + 4 * (d + 1)


def index_keys(keys: torch.Tensor) -> KeyIndex:
    """Stable (key, row) sort + run bounds of an int64 key column.

    Replaces tensorpath.py:78-93 (to_tensor): positions = stable argsort,
    key_values = distinct keys, offsets = CSR run starts + [n].
    """
    _require_cuda(keys, "keys")
    if keys.dtype != torch.int64 or keys.dim() != 1:
        raise ValueError("keys must be a 1-D int64 tensor")
    keys = aligned16(keys)
    lib = C.load()
    n = keys.numel()
    dev = keys.device
    s = stream_handle()
    positions = torch.empty(n, dtype=_U32, device=dev)
    key_values = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    offsets = torch.empty(n + 1, dtype=_U32, device=dev)
    d = torch.empty(1, dtype=torch.int64, device=dev)
    if n > 0:
        sorted_keys = torch.empty(n, dtype=torch.int64, device=dev)
        ws_bytes = lib.rl_sort_workspace_bytes(n)
        ws = workspace(ws_bytes, dev)
        C.check(
            lib.rl_sort_axis(_ptr(keys), C.RL_COL_INT64, 8, 0, 0, None, n, _ptr(sorted_keys), _ptr(positions),
                             _ptr(ws), ws.numel(), s),
            "rl_sort_axis",
        )
        del ws
        rb_ws = workspace(lib.rl_run_bounds_workspace_bytes(n), dev)
        C.check(
            lib.rl_run_bounds(_ptr(sorted_keys), n, _ptr(key_values), _ptr(offsets), _ptr(d), _ptr(rb_ws),
                              rb_ws.numel(), s),
            "rl_run_bounds",
        )
    else:
        rb_ws = workspace(lib.rl_run_bounds_workspace_bytes(0), dev)
        C.check(lib.rl_run_bounds(_ptr(keys), 0, _ptr(key_values), _ptr(offsets), _ptr(d), _ptr(rb_ws),
                                  rb_ws.numel(), s), "rl_run_bounds")
    return KeyIndex(n, key_values, offsets, positions, d)


@dataclass
class Alignment:
    """Matched keys of two key axes + join sizing, on the device."""

    cap: int
    matched_keys: torch.Tensor  # int64 [cap]
    left_starts: torch.Tensor  # uint32 bits [cap]
    left_counts: torch.Tensor
    right_starts: torch.Tensor
    right_counts: torch.Tensor
    pair_offsets: torch.Tensor  # uint64 bits (int64 tensor) [cap + 1]
    m_total: torch.Tensor  # int64 [2]: M, total pairs (device scalars)


def align(left: KeyIndex, right: KeyIndex) -> Alignment:
    """K4+K5: key_axis_align + per-key pair counts and their exclusive scan
    (tensorpath.py:109-128, 149-161), no host synchronisation."""
    lib = C.load()
    dev = left.positions.device
    cap = min(left.n, right.n)
    alloc = max(cap, 1)
    mk = torch.empty(alloc, dtype=torch.int64, device=dev)
    ls = torch.empty(alloc, dtype=_U32, device=dev)
    lc = torch.empty(alloc, dtype=_U32, device=dev)
    rs = torch.empty(alloc, dtype=_U32, device=dev)
    rc = torch.empty(alloc, dtype=_U32, device=dev)
    po = torch.empty(alloc + 1, dtype=torch.int64, device=dev)
    mt = torch.empty(2, dtype=torch.int64, device=dev)
    grid_cap = left.n if cap > 0 else 0
    ws = workspace(lib.rl_align_workspace_bytes(grid_cap), dev)
    C.check(
        lib.rl_key_axis_align(
            _ptr(left.key_values), _ptr(left.offsets), _ptr(left.d), grid_cap,
            _ptr(right.key_values), _ptr(right.offsets), _ptr(right.d),
            _ptr(mk), _ptr(ls), _ptr(lc), _ptr(rs), _ptr(rc), _ptr(po),
            ctypes.c_void_p(mt.data_ptr()), ctypes.c_void_p(mt.data_ptr() + 8),
            _ptr(ws), ws.numel(), stream_handle(),
        ),
        "rl_key_axis_align",
    )
    return Alignment(cap, mk, ls, lc, rs, rc, po, mt)


def fetch_scalars(*tensors: torch.Tensor) -> list:
    """One pinned D2H of several small device int64 tensors, one sync."""
    flat = [t.reshape(-1) for t in tensors]
    total = sum(t.numel() for t in flat)
    host = torch.empty(total, dtype=torch.int64, pin_memory=True)
    off = 0
    for t in flat:
        host[off : off + t.numel()].copy_(t, non_blocking=True)
        off += t.numel()
    torch.cuda.current_stream().synchronize()
    return host.tolist()


@dataclass
class OutColumn:
    """One output column of a join/gather: dst[t] = src[row(t)]."""

    src: Optional[torch.Tensor]  # device rows × width bytes (None for the key column)
    dst: torch.Tensor  # device
    width: int
    side: int  # C.RL_SIDE_*


def expand(
    al: Alignment,
    m: int,
    left: KeyIndex,
    right: KeyIndex,
    out_begin: int,
    out_end: int,
    columns: Sequence[OutColumn] = (),
    left_rows: Optional[torch.Tensor] = None,
    right_rows: Optional[torch.Tensor] = None,
) -> None:
    """K6+K7: materialise output pairs [out_begin, out_end) in reference
    order (key, left row, right row) and gather the columns in one pass."""
    lib = C.load()
    arr, ncols = C.columns_array(
        (None if c.src is None else c.src.data_ptr(), c.dst.data_ptr(), c.width, c.side) for c in columns
    )
    C.check(
        lib.rl_join_expand(
            _ptr(al.matched_keys), _ptr(al.left_starts), _ptr(al.right_starts), _ptr(al.right_counts),
            _ptr(al.pair_offsets), m, _ptr(left.positions), _ptr(right.positions), out_begin, out_end,
            _ptr(left_rows), _ptr(right_rows), arr, ncols, stream_handle(),
        ),
        "rl_join_expand",
    )


def pair_checksum(al: Alignment, m: int, left: KeyIndex, right: KeyIndex, out_begin: int, out_end: int,
                  acc: torch.Tensor) -> None:
    """Accumulate sum(fmix64(l << 32 | r)) over pairs [out_begin, out_end) into acc (int64[1])."""
    lib = C.load()
    C.check(
        lib.rl_join_pair_checksum(
            _ptr(al.left_starts), _ptr(al.right_starts), _ptr(al.right_counts), _ptr(al.pair_offsets), m,
            _ptr(left.positions), _ptr(right.positions), out_begin, out_end, _ptr(acc), stream_handle(),
        ),
        "rl_join_pair_checksum",
    )


@dataclass
class SortAxis:
    """One sort key on the device: int64 [n] or uint8 [n, w] (Bytes(w))."""

    data: torch.Tensor
    descending: bool = False

    @property
    def is_int64(self) -> bool:
        return self.data.dtype == torch.int64 and self.data.dim() == 1


def sort_permutation(axes: Sequence[SortAxis], n: int, device, sorted_keys_out: Optional[torch.Tensor] = None,
                     gather: Sequence[OutColumn] = (), fuse_gather: bool = False) -> torch.Tensor:
    """Stable multi-key order: LSD over the key axes, least significant first
    (tensorpath.py:243-246); Bytes axes go word by word from the last word
    (tensorpath.py:226-228). Returns the permutation (uint32 bits, int32).

    sorted_keys_out (optional) receives the sorted values of the single
    int64 key when there is exactly one key axis (the cfg2 ORDER BY).
    gather: columns taken by the final permutation (Relation.take): one
    gather launch after the sort, or, with fuse_gather and at most 8
    columns, inside the last digit pass. Measured on B200 (cfg2, 10M rows,
    4-byte payload): the separate launch takes 55 us, the fused variant adds
    ~165 us to the last pass (its random payload reads contend with the
    pass's streaming traffic for L2 at 2 CTAs/SM), so fusion is opt-in.
    """
    lib = C.load()
    s = stream_handle()
    perm: Optional[torch.Tensor] = None
    if n == 0:
        return torch.empty(0, dtype=_U32, device=device)
    ws = workspace(lib.rl_sort_workspace_bytes(n), device)
    if sorted_keys_out is not None and not (len(axes) == 1 and axes[0].is_int64):
        raise ValueError("sorted_keys_out needs exactly one int64 key axis")
    gather = list(gather)
    fuse = fuse_gather and 0 < len(gather) <= C.RL_SORT_MAX_FUSED_COLUMNS
    steps = []
    for axis in reversed(list(axes)):
        _require_cuda(axis.data, "sort axis")
        data = aligned16(axis.data)
        if axis.is_int64:
            steps += [(axis, data, C.RL_COL_INT64, 8, 0)]
        else:
            w = axis.data.shape[1]
            steps += [(axis, data, C.RL_COL_BYTES, w, j) for j in range(max(1, -(-w // 8)) - 1, -1, -1)]
    if fuse and steps[-1][3] == 0:  # a zero-width final word has no pass to fuse into
        fuse = False
    for i, (axis, data, kind, width, word) in enumerate(steps):
        out = torch.empty(n, dtype=_U32, device=device)
        keys_out = _ptr(sorted_keys_out) if perm is None and kind == C.RL_COL_INT64 else None
        if fuse and i == len(steps) - 1:
            arr, ncols = C.columns_array((c.src.data_ptr(), c.dst.data_ptr(), c.width, C.RL_SIDE_LEFT) for c in gather)
            st = lib.rl_sort_axis_gather(_ptr(data), kind, width, word, int(axis.descending), _ptr(perm), n,
                                         keys_out, _ptr(out), arr, ncols, _ptr(ws), ws.numel(), s)
        else:
            st = lib.rl_sort_axis(_ptr(data), kind, width, word, int(axis.descending), _ptr(perm), n, keys_out,
                                  _ptr(out), _ptr(ws), ws.numel(), s)
        C.check(st, "rl_sort_axis")
        perm = out
    if gather and not fuse:
        gather_rows(perm, gather)
    return perm


CARRY_MIN_ROWS = 4 << 20  # the scatter path (below it the plain sort + gather is used anyway)


def packable_keys(keys: torch.Tensor, samples: int = 4096) -> bool:
    """Whether the int64 keys probably vary in at most 32 bits in at most two
    runs (the scatter path's packed rows, radix_sort.cu pack_code_of): the OR
    of (key ^ first key) over strided samples (one small D2H). A bit the
    sample misses is caught on the device (the sort then takes the LSD
    passes with the gathers fused — correct, only slower)."""
    import numpy as np

    n = keys.numel()
    if n == 0:
        return False
    v = keys[:: max(1, n // samples)].cpu().numpy().view(np.uint64)
    vary = int(np.bitwise_or.reduce(v ^ v[0]))
    bits = [(vary >> b) & 1 for b in range(64)]
    runs = sum(1 for b in range(64) if bits[b] and (b == 63 or not bits[b + 1]))
    return vary != 0 and runs <= 2 and sum(bits) <= 32


def sort_carry(keys: torch.Tensor, descending: bool, sorted_keys_out: Optional[torch.Tensor],
               columns: Sequence[OutColumn]) -> torch.Tensor:
    """ORDER BY one int64 key with every other column carried with the rows
    (rl_sort_axis_carry): dst row o = src row perm[o]. Returns the permutation."""
    lib = C.load()
    keys = aligned16(keys)
    n = keys.numel()
    perm = torch.empty(n, dtype=_U32, device=keys.device)
    if n == 0:
        return perm
    arr, ncols = C.columns_array((c.src.data_ptr(), c.dst.data_ptr(), c.width, C.RL_SIDE_LEFT) for c in columns)
    ws = workspace(lib.rl_sort_carry_workspace_bytes(n, sum(c.width for c in columns)), keys.device)
    C.check(lib.rl_sort_axis_carry(_ptr(keys), n, int(descending), _ptr(sorted_keys_out), _ptr(perm), arr, ncols,
                                   _ptr(ws), ws.numel(), stream_handle()), "rl_sort_axis_carry")
    return perm


def carry_fits(columns: Sequence[OutColumn]) -> bool:
    """<= 4 columns of <= 16 bytes a row together (natural alignment)."""
    if not 0 < len(columns) <= 4:
        return False
    at = 0
    for w in sorted((c.width for c in columns), reverse=True):
        al = 8 if w % 8 == 0 else 4 if w % 4 == 0 else 1
        at = -(-at // al) * al + w
    return at <= 16


def idw_fits(columns: Sequence[OutColumn]) -> bool:
    """<= 4 carried bytes a row: on keys that do not pack they share one word
    with the row id through the sort's passes (radix_sort.cu, idw), 16 bytes a
    row instead of 12 + a random gather afterwards."""
    return 0 < len(columns) <= 4 and sum(c.width for c in columns) <= 4


class SortGraph:
    """A stable ORDER BY of one int64 key column (+ Relation.take of bound
    columns) captured once as a CUDA graph: histogram, cooperative sort and
    gather replay without host launch work (repeated sorts of same-shaped,
    device-resident inputs — e.g. a serving loop). ``replay()`` sorts the
    current contents of ``keys`` / the gather sources into ``sorted_keys``,
    ``perm`` and the gather destinations, which are fixed at capture."""

    def __init__(self, keys: torch.Tensor, descending: bool = False, gather: Sequence[OutColumn] = (),
                 carry: Optional[bool] = None):
        """carry: move the gathered columns with the rows through the sort's
        passes (rl_sort_axis_carry) instead of gathering them by the
        permutation afterwards; None = RL_SORT_CARRY=1 (off by default: for
        cfg2 the gather is as fast)."""
        _require_cuda(keys, "keys")
        lib = C.load()
        self.keys = aligned16(keys)
        n = self.keys.numel()
        dev = self.keys.device
        self.sorted_keys = torch.empty(n, dtype=torch.int64, device=dev)
        self.perm = torch.empty(n, dtype=_U32, device=dev)
        self.gather = list(gather)
        if carry is None:
            env = os.environ.get("RL_SORT_CARRY", "")
            # measured at cfg2 (10M rows, 4-byte payload): carried 0.308 ms a step vs
            # 0.302 sort + gather, so the gather stays the default
            carry = env == "1"
        self.carry = bool(carry and self.gather)
        if self.carry:
            arr, ncols = C.columns_array((c.src.data_ptr(), c.dst.data_ptr(), c.width, C.RL_SIDE_LEFT)
                                         for c in self.gather)
            self._cols = (arr, ncols)
            self._ws = workspace(lib.rl_sort_carry_workspace_bytes(n, sum(c.width for c in self.gather)), dev)
        else:
            self._ws = workspace(lib.rl_sort_workspace_bytes(n), dev)
        self._desc = int(descending)

        def body():
            if self.carry:
                C.check(lib.rl_sort_axis_carry(_ptr(self.keys), n, self._desc, _ptr(self.sorted_keys),
                                               _ptr(self.perm), self._cols[0], self._cols[1], _ptr(self._ws),
                                               self._ws.numel(), stream_handle()), "rl_sort_axis_carry")
                return
            C.check(lib.rl_sort_axis(_ptr(self.keys), C.RL_COL_INT64, 8, 0, self._desc, None, n,
                                     _ptr(self.sorted_keys), _ptr(self.perm), _ptr(self._ws), self._ws.numel(),
                                     stream_handle()), "rl_sort_axis")
            if self.gather:
                gather_rows(self.perm, self.gather)

        side = torch.cuda.Stream(device=dev)  # warm-up outside the capture (lazy attributes, allocator)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            body()
        torch.cuda.current_stream(dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        c0 = lib.rl_launch_count()
        with torch.cuda.graph(self.graph):
            body()
        self.launches_per_replay = lib.rl_launch_count() - c0

    def replay(self) -> None:
        self.graph.replay()


def gather_rows(rows: torch.Tensor, columns: Sequence[OutColumn]) -> None:
    """K7: dst row t = src row rows[t] for every column (Relation.take)."""
    lib = C.load()
    arr, ncols = C.columns_array((c.src.data_ptr(), c.dst.data_ptr(), c.width, C.RL_SIDE_LEFT) for c in columns)
    C.check(lib.rl_gather_rows(_ptr(rows), rows.numel(), arr, ncols, stream_handle()), "rl_gather_rows")


def gather_split16(rows: torch.Tensor, src16: torch.Tensor, dst_lo: torch.Tensor, dst_hi: torch.Tensor) -> None:
    """Relation.take of two 8-byte columns stored row-interleaved (src16: rows
    of 16 bytes): one random 16-byte load a row into two column outputs."""
    C.check(C.load().rl_gather_rows_split16(_ptr(rows), rows.numel(), _ptr(src16), _ptr(dst_lo), _ptr(dst_hi),
                                            stream_handle()), "rl_gather_rows_split16")


def widen(u32: torch.Tensor, n: Optional[int] = None) -> torch.Tensor:
    """uint32 bits → int64 values (positions/offsets handed back as int64)."""
    lib = C.load()
    n = u32.numel() if n is None else n
    out = torch.empty(n, dtype=torch.int64, device=u32.device)
    C.check(lib.rl_widen_u32(_ptr(u32), n, _ptr(out), stream_handle()), "rl_widen_u32")
    return out


def hash_partition(keys: torch.Tensor, parts: int, seed: int, columns: Sequence[OutColumn] = ()):
    """K8: stable hash partition by hash_i64(key, seed) % parts
    (hashing.py:54-61). Returns (row ids grouped by destination, counts[parts])."""
    lib = C.load()
    n = keys.numel()
    dev = keys.device
    rows = torch.empty(n, dtype=_U32, device=dev)
    counts = torch.empty(parts, dtype=torch.int64, device=dev)
    ws = workspace(lib.rl_partition_workspace_bytes(n, parts), dev)
    arr, ncols = C.columns_array((c.src.data_ptr(), c.dst.data_ptr(), c.width, C.RL_SIDE_LEFT) for c in columns)
    C.check(
        lib.rl_hash_partition(_ptr(keys), n, parts, seed & (2**64 - 1), arr, ncols, _ptr(rows), _ptr(counts),
                              _ptr(ws), ws.numel(), stream_handle()),
        "rl_hash_partition",
    )
    return rows, counts


def range_partition(keys: torch.Tensor, gid_base: int, split_keys: torch.Tensor, split_gids: torch.Tensor,
                    descending: bool = False, columns: Sequence[OutColumn] = ()):
    """K8 (sort variant): stable range partition by (key, global row id)
    against sorted splitters. Returns (row ids grouped by destination,
    counts[len(splitters) + 1])."""
    lib = C.load()
    n = keys.numel()
    dev = keys.device
    parts = split_keys.numel() + 1
    rows = torch.empty(n, dtype=_U32, device=dev)
    counts = torch.empty(parts, dtype=torch.int64, device=dev)
    ws = workspace(lib.rl_partition_workspace_bytes(n, parts), dev)
    sk = split_keys.to(device=dev, dtype=torch.int64).contiguous()
    sg = split_gids.to(device=dev, dtype=torch.int64).contiguous()
    arr, ncols = C.columns_array((c.src.data_ptr(), c.dst.data_ptr(), c.width, C.RL_SIDE_LEFT) for c in columns)
    C.check(
        lib.rl_range_partition(_ptr(keys.contiguous()), n, int(gid_base), _ptr(sk), _ptr(sg), parts - 1,
                               int(descending), arr, ncols, _ptr(rows), _ptr(counts), _ptr(ws), ws.numel(),
                               stream_handle()),
        "rl_range_partition",
    )
    return rows, counts


def multiset_digest(columns: Sequence[torch.Tensor]) -> int:
    """The reference's 128-bit multiset digest (relation.py:319-330) of the
    relation whose columns (schema order; int64 [n] or uint8 [n, w]) are on
    the device. Returns the 128-bit int (0 for an empty relation)."""
    lib = C.load()
    cols = [c.contiguous() for c in columns]
    if not cols:
        raise ValueError("a relation has at least one column")
    n = cols[0].shape[0]
    arr, ncols = C.columns_array(
        (c.data_ptr(), None, c.element_size() * (c.shape[1] if c.dim() > 1 else 1), C.RL_SIDE_LEFT) for c in cols
    )
    out = torch.empty(2, dtype=torch.int64, device=cols[0].device)
    C.check(lib.rl_multiset_digest(arr, ncols, n, _ptr(out), stream_handle()), "rl_multiset_digest")
    hi, lo = (int(v) & (2**64 - 1) for v in fetch_scalars(out))
    return (hi << 64) | lo


BJ_MIN_ROWS = 4 << 20  # smaller joins: the sort-based plan (fewer launches; measured crossover ~4M rows a side)
BJ_CARRY_MIN_RATIO = 0.5  # carry payloads when the expected pairs reach half the larger side (measured break-even)


def _bjoin_allowed(nl: int, nr: int) -> bool:
    import os

    if os.environ.get("RL_NO_BJOIN", "") not in ("", "0"):
        return False
    if os.environ.get("RL_FORCE_BJOIN", "") not in ("", "0"):
        return nl >= 1 and nr >= 1
    return min(nl, nr) >= BJ_MIN_ROWS and max(nl, nr) <= C.RL_MAX_ROWS


class BucketJoinPlan:
    """rl_bjoin_plan_build result (csrc/bucket_join.cu): both sides as packed
    (key | row id) words in the same 65536 sub-buckets, the pairs counted per
    run on chip and scanned; no sorted key axes. ``applies`` is False when the
    keys need more than 32 bits or a sub-bucket is too large (skew) — then
    use JoinPlanDev. Same expand / pair_checksum contract as JoinPlanDev."""

    kind = "bucket"

    def __init__(self, left_keys: torch.Tensor, right_keys: torch.Tensor, left_carry: Sequence[torch.Tensor] = (),
                 right_carry: Sequence[torch.Tensor] = ()):
        """left_carry / right_carry: the columns whose output copies expand
        will gather (the join's non-key columns) — carried with the rows
        through the partition passes (<= 16 bytes a row a side) so that expand
        reads them beside the row instead of at random row ids."""
        lib = C.load()
        lk, rk = aligned16(left_keys), aligned16(right_keys)
        self._keys = (lk, rk)  # the plan reads the left keys again in expand (constant key bits)
        import os

        if os.environ.get("RL_BJ_NO_CARRY", "") not in ("", "0"):  # A/B: gather every column by row id
            left_carry, right_carry = (), ()
        self._carry = (list(left_carry), list(right_carry))  # kept alive: expand matches their pointers
        nl, nr = lk.numel(), rk.numel()
        arrs = [C.columns_array((c.data_ptr(), None, c.element_size() * (c.shape[1] if c.dim() > 1 else 1),
                                 C.RL_SIDE_LEFT) for c in side) for side in self._carry]
        words = [lib.rl_bjoin_carry_words(arr, n) if n else 0 for arr, n in arrs]
        self.ws = workspace(lib.rl_bjoin_workspace_bytes(nl, nr, max(words[0], 0), max(words[1], 0)), lk.device)
        self.plan = C.RlBjoinPlan()
        C.check(lib.rl_bjoin_plan_build(_ptr(lk), nl, _ptr(rk), nr, arrs[0][0], arrs[0][1], arrs[1][0], arrs[1][1],
                                        _ptr(self.ws), self.ws.numel(), ctypes.byref(self.plan), stream_handle()),
                "rl_bjoin_plan_build")
        self.n_left, self.n_right = nl, nr
        host = torch.empty(2, dtype=torch.int64, pin_memory=True)
        off = self.plan.scalars - self.ws.data_ptr()
        host.view(torch.uint8).copy_(self.ws[off : off + 16], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self.total, ok = host.tolist()
        self.applies = bool(ok)

    def expand(self, out_begin: int, out_end: int, columns: Sequence[OutColumn] = (),
               left_rows: Optional[torch.Tensor] = None, right_rows: Optional[torch.Tensor] = None,
               dst_strides: Optional[Sequence[int]] = None) -> None:
        """dst_strides: bytes between output rows per column (None / 0 = the
        width) — 8- or 16-byte columns written row-interleaved into one buffer."""
        lib = C.load()
        arr, ncols = C.columns_array(
            (None if c.src is None else c.src.data_ptr(), c.dst.data_ptr(), c.width, c.side) for c in columns
        )
        if dst_strides is None:
            C.check(lib.rl_bjoin_expand(ctypes.byref(self.plan), out_begin, out_end, _ptr(left_rows),
                                        _ptr(right_rows), arr, ncols, stream_handle()), "rl_bjoin_expand")
            return
        st = (ctypes.c_int32 * max(1, len(columns)))(*[int(x or 0) for x in dst_strides])
        C.check(lib.rl_bjoin_expand_strided(ctypes.byref(self.plan), out_begin, out_end, _ptr(left_rows),
                                            _ptr(right_rows), arr, ncols, st, stream_handle()),
                "rl_bjoin_expand_strided")

    def pair_checksum(self, out_begin: int, out_end: int, acc: torch.Tensor) -> None:
        C.check(C.load().rl_bjoin_pair_checksum(ctypes.byref(self.plan), out_begin, out_end, _ptr(acc),
                                                stream_handle()), "rl_bjoin_pair_checksum")


def expected_pairs_ratio(left_keys: torch.Tensor, right_keys: torch.Tensor, samples: int = 2048) -> float:
    """Pairs per row of the larger side a join of uniform keys would produce:
    nl * nr / (key range) / max(nl, nr), the range taken from strided samples
    of both sides (one small reduction, one host sync). Carrying payload
    through the bucket join's passes costs ~2 passes x 2 x width per input
    row and saves ~2 random sector reads per output pair: it pays when pairs
    are about as many as rows (cfg5), not for selective joins (cfg4: ~0.02)."""
    nl, nr = left_keys.numel(), right_keys.numel()
    s = torch.cat([left_keys[:: max(1, nl // samples)], right_keys[:: max(1, nr // samples)]])
    lo, hi = (int(v) for v in torch.aminmax(s))
    rng = max(1, hi - lo + 1)
    return nl * nr / rng / max(nl, nr, 1)


def plan_join(left_keys: torch.Tensor, right_keys: torch.Tensor, left_carry: Sequence[torch.Tensor] = (),
              right_carry: Sequence[torch.Tensor] = ()):
    """The join plan for two int64 key columns on the device: the bucket join
    when it applies (<= 32 varying key bits, no oversized sub-bucket; the
    carry columns ride with the rows), else the sort-based plan (both key
    axes + alignment). One host sync either way (plus one when the bucket
    join declines)."""
    if _bjoin_allowed(left_keys.numel(), right_keys.numel()):
        if (left_carry or right_carry) and expected_pairs_ratio(left_keys, right_keys) < BJ_CARRY_MIN_RATIO:
            left_carry, right_carry = (), ()  # selective join: gather the few output rows by row id instead
        bp = BucketJoinPlan(left_keys, right_keys, left_carry, right_carry)
        if bp.applies:
            return bp
        del bp
    return JoinPlanDev(left_keys, right_keys)


class JoinPlanDev:
    """rl_join_plan_build result: both key axes indexed and aligned inside
    one workspace (device pointers in ``plan``), totals fetched once."""

    kind = "sort"

    def __init__(self, left_keys: torch.Tensor, right_keys: torch.Tensor):
        lib = C.load()
        lk, rk = aligned16(left_keys), aligned16(right_keys)
        nl, nr = lk.numel(), rk.numel()
        self.ws = workspace(lib.rl_join_plan_workspace_bytes(nl, nr), lk.device)
        self.plan = C.RlJoinPlan()
        C.check(lib.rl_join_plan_build(_ptr(lk), nl, _ptr(rk), nr, _ptr(self.ws), self.ws.numel(),
                                       ctypes.byref(self.plan), stream_handle()), "rl_join_plan_build")
        self.n_left, self.n_right = nl, nr
        # one pinned D2H of the device scalars (D_left, D_right, M, total) + one sync
        off = self.plan.scalars - self.ws.data_ptr()
        host = torch.empty(4, dtype=torch.int64, pin_memory=True)
        host.view(torch.uint8).copy_(self.ws[off : off + 32], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self.d_left, self.d_right, self.matched_keys, self.total = host.tolist()

    def expand(self, out_begin: int, out_end: int, columns: Sequence[OutColumn] = (),
               left_rows: Optional[torch.Tensor] = None, right_rows: Optional[torch.Tensor] = None) -> None:
        lib = C.load()
        p = self.plan
        arr, ncols = C.columns_array(
            (None if c.src is None else c.src.data_ptr(), c.dst.data_ptr(), c.width, c.side) for c in columns
        )
        C.check(lib.rl_join_expand(p.matched_keys, p.left_starts, p.right_starts, p.right_counts, p.pair_offsets,
                                   self.matched_keys, p.left_positions, p.right_positions, out_begin, out_end,
                                   _ptr(left_rows), _ptr(right_rows), arr, ncols, stream_handle()),
                "rl_join_expand")

    def pair_checksum(self, out_begin: int, out_end: int, acc: torch.Tensor) -> None:
        lib = C.load()
        p = self.plan
        C.check(lib.rl_join_pair_checksum(p.left_starts, p.right_starts, p.right_counts, p.pair_offsets,
                                          self.matched_keys, p.left_positions, p.right_positions, out_begin,
                                          out_end, _ptr(acc), stream_handle()), "rl_join_pair_checksum")
