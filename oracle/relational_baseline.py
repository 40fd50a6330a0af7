"""CPU RELATIONAL baseline: the reference's memory-budgeted Grace hash join
with temp-file spill, restated in numpy — TEST / BASELINE INFRASTRUCTURE ONLY.

The north star (BASELINE.json) asks for the reference's CPU relational
hash-join path (work_mem = 1 MB, spill blocks / temp MB counted) to be timed
on the GPU box's own host cores beside the B200 path. The reference package
does not travel to the box, so this module restates it: only `bench.py`'s
baseline leg and `tests/` use it, never the product path.

Restated from /root/reference/pkg/src/relab:
  rowpath.py:25-32   constants (JOIN_BASE_SEED, reseed multiplier, bucket salt,
                     MAX_RECURSION 8, MAX_FANOUT 1024)
  rowpath.py:56-91   _bucket_pairs (power-of-two buckets, load <= 0.5)
  rowpath.py:177-233 hash_join_row (in-memory when the build side fits the
                     budget, else Grace partitioning); build side = the
                     smaller serialized input
  rowpath.py:265-307 _join_partitioned (fanout min(1024, ceil(est/budget)+1),
                     per-pair recursion under a reseeded hash)
  rowpath.py:310-335 _spill_partitions (hash % fanout, one stream per
                     non-empty partition)
  spill.py:21-23, 112-158, 200-232  8 KiB blocks with a 2-byte used-length
                     header, zero padded; spill_rows / read_stream_matrix
  relation.py:138-151 canonical row serialisation
  hashing.py:32-61   fmix64 / hash_i64
Pinned against the live reference by tests/test_relational_baseline.py
(temp block counts and the output multiset).
"""

from __future__ import annotations

import os
import shutil
import tempfile
from dataclasses import dataclass

import numpy as np

from .tensorpath_oracle import fmix64, fmix64_scalar

JOIN_BASE_SEED = 0x9E3779B97F4A7C15
RESEED_MULT = 0x2545F4914F6CDD1D
BUCKET_SALT = 0x6A09E667F3BCC909
MAX_RECURSION = 8
MAX_FANOUT = 1024
BLOCK_SIZE = 8192
BLOCK_HEADER = 2
BLOCK_CAPACITY = BLOCK_SIZE - BLOCK_HEADER
M64 = (1 << 64) - 1


def hash_i64(keys: np.ndarray, seed: int) -> np.ndarray:
    u = np.ascontiguousarray(keys, dtype=np.int64).view(np.uint64)
    return fmix64(u ^ np.uint64(fmix64_scalar(seed)))


@dataclass
class SpillCounts:
    temp_blocks_written: int = 0
    temp_bytes_written: int = 0
    temp_bytes_read: int = 0
    partition_passes: int = 0

    @property
    def temp_mb(self) -> float:
        return self.temp_blocks_written * BLOCK_SIZE / 2**20


class Arena:
    """Temp streams of fixed-width rows in zero-padded 8 KiB blocks."""

    def __init__(self, directory=None):
        self.root = tempfile.mkdtemp(prefix="relarena-", dir=directory)
        self.stats = SpillCounts()
        self.n = 0

    def close(self):
        shutil.rmtree(self.root, ignore_errors=True)

    def spill(self, rows: np.ndarray) -> str:
        n, width = rows.shape
        rpb = BLOCK_CAPACITY // width
        nb = -(-n // rpb)
        buf = np.zeros((nb, BLOCK_SIZE), dtype=np.uint8)
        padded = np.zeros((nb * rpb, width), dtype=np.uint8)
        padded[:n] = rows
        buf[:, BLOCK_HEADER:BLOCK_HEADER + rpb * width] = padded.reshape(nb, rpb * width)
        used = np.full(nb, rpb * width, dtype=np.uint16)
        used[-1] = (n - (nb - 1) * rpb) * width
        buf[:, 0] = (used & 0xFF).astype(np.uint8)
        buf[:, 1] = (used >> 8).astype(np.uint8)
        path = os.path.join(self.root, f"s{self.n:05d}.tmp")
        self.n += 1
        with open(path, "wb") as f:
            f.write(buf.reshape(-1).data)
        self.stats.temp_blocks_written += nb
        self.stats.temp_bytes_written += nb * BLOCK_SIZE
        return path + f"|{width}"

    def read(self, sid: str) -> np.ndarray:
        path, width = sid.rsplit("|", 1)
        width = int(width)
        blocks = np.fromfile(path, dtype=np.uint8).reshape(-1, BLOCK_SIZE)
        self.stats.temp_bytes_read += blocks.size
        used = blocks[:, 0].astype(np.int64) | (blocks[:, 1].astype(np.int64) << 8)
        rpb = BLOCK_CAPACITY // width
        region = np.ascontiguousarray(blocks[:, BLOCK_HEADER:BLOCK_HEADER + rpb * width]).reshape(-1, width)
        return region[: int((used // width).sum())]


def bucket_pairs(build_keys, probe_keys, seed):
    nb, npr = len(build_keys), len(probe_keys)
    empty = np.empty(0, dtype=np.int64)
    if nb == 0 or npr == 0:
        return empty, empty
    size = 1 << max(3, (2 * nb - 1).bit_length())
    mask = np.uint64(size - 1)
    dt = np.int32 if size <= 2**31 else np.int64
    hb = (hash_i64(build_keys, seed) & mask).astype(dt)
    grouped = np.argsort(hb, kind="quicksort")
    counts = np.bincount(hb, minlength=size)
    starts = np.zeros(size + 1, dtype=np.int64)
    np.cumsum(counts, out=starts[1:])
    hp = (hash_i64(probe_keys, seed) & mask).astype(dt)
    cc = counts[hp]
    total = int(cc.sum())
    if total == 0:
        return empty, empty
    cum = np.zeros(npr + 1, dtype=np.int64)
    np.cumsum(cc, out=cum[1:])
    within = np.arange(total, dtype=np.int64) - np.repeat(cum[:-1], cc)
    cand = np.repeat(starts[hp], cc) + within
    br = grouped[cand]
    pr = np.repeat(np.arange(npr, dtype=np.int64), cc)
    eq = build_keys[br] == probe_keys[pr]
    return br[eq], pr[eq]


def serialize(cols, widths) -> np.ndarray:
    n = len(cols[0])
    out = np.empty((n, sum(widths)), dtype=np.uint8)
    off = 0
    for c, w in zip(cols, widths):
        if c.dtype == np.int64:
            out[:, off:off + 8] = c.astype("<i8", copy=False).view(np.uint8).reshape(n, 8)
        elif w:
            out[:, off:off + w] = c
        off += w
    return out


def _keys(mat, off):
    return np.ascontiguousarray(mat[:, off:off + 8]).view("<i8").ravel()


def hash_join_row(left_cols, left_widths, left_key, right_cols, right_widths, right_key,
                  budget_bytes: int = 1 << 20, temp_dir=None):
    """rowpath.hash_join_row: returns (number of output rows, SpillCounts).
    Output rows are materialised (serialized) like the reference's."""
    lbytes = len(left_cols[0]) * sum(left_widths)
    rbytes = len(right_cols[0]) * sum(right_widths)
    build_left = lbytes <= rbytes
    b_cols, b_w, b_k = (left_cols, left_widths, left_key) if build_left else (right_cols, right_widths, right_key)
    p_cols, p_w, p_k = (right_cols, right_widths, right_key) if build_left else (left_cols, left_widths, left_key)
    b_width, p_width = sum(b_w), sum(p_w)
    b_off, p_off = sum(b_w[:b_k]), sum(p_w[:p_k])
    arena = Arena(temp_dir)
    out_rows = [0]
    chunks = []

    def emit(bm, pm, bi, pi):
        if len(bi) == 0:
            return
        chunks.append(np.concatenate([bm[bi], pm[pi]], axis=1))  # the same bytes moved as the reference
        out_rows[0] += len(bi)

    def join_part(bm, bk, pm, pk, depth, seed):
        est = bm.shape[0] * b_width
        if est <= budget_bytes:
            bi, pi = bucket_pairs(bk, pk, seed ^ BUCKET_SALT)
            emit(bm, pm, bi, pi)
            return
        if depth >= MAX_RECURSION:
            raise RuntimeError("build partition still exceeds the budget after 8 levels")
        fanout = min(MAX_FANOUT, -(-est // budget_bytes) + 1)
        arena.stats.partition_passes += 1

        def spill_side(mat, keys):
            part = (hash_i64(keys, seed) % np.uint64(fanout)).astype(np.int32)
            order = np.argsort(part, kind="quicksort")
            bounds = np.searchsorted(part[order], np.arange(fanout + 1, dtype=np.int32))
            ids = []
            for p in range(fanout):
                lo, hi = int(bounds[p]), int(bounds[p + 1])
                ids.append(None if lo == hi else arena.spill(mat[order[lo:hi]]))
            return ids

        bids, pids = spill_side(bm, bk), spill_side(pm, pk)
        child = (seed * RESEED_MULT + depth + 1) & M64
        for bid, pid in zip(bids, pids):
            if bid is None or pid is None:
                continue
            b2, p2 = arena.read(bid), arena.read(pid)
            join_part(b2, _keys(b2, b_off), p2, _keys(p2, p_off), depth + 1, child)

    try:
        if len(b_cols[0]) * b_width <= budget_bytes:
            bi, pi = bucket_pairs(b_cols[b_k], p_cols[p_k], JOIN_BASE_SEED ^ BUCKET_SALT)
            out_rows[0] = len(bi)
            _ = [c[bi] for c in b_cols] + [c[pi] for c in p_cols]
        else:
            bm, pm = serialize(b_cols, b_w), serialize(p_cols, p_w)
            join_part(bm, _keys(bm, b_off), pm, _keys(pm, p_off), 0, JOIN_BASE_SEED)
            if chunks:
                np.concatenate(chunks)
    finally:
        arena.close()
    return out_rows[0], arena.stats
