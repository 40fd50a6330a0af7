"""Multi-GPU tensor path: one process per GPU, one exchange step per operator.

North star / SURVEY.md §8(e): inputs shard naturally. Each rank holds a
contiguous global row range of every relation (rank r owns rows
[base_r, base_r + n_r)), so global row ids are base + local row.

* Join: every rank hash-partitions R and S by ``hash_i64(key, seed) % P``
  (hashing.py:54-61) with the stable device partition (K8), exchanges the
  per-destination counts and then (key, global row id, payload columns) with
  ``all_to_all_single`` (NCCL over NVLink on GPUs), and joins locally with
  K1-K7. A key lands on exactly one rank; rows arrive grouped by source rank
  in source order, i.e. in ascending global row id, so the local stable join
  emits every key's pairs in the reference's (left row, right row) order.
  The match count is an all-reduce SUM. Output stays sharded.
* ORDER BY: regular samples of (key, global row id) are all-gathered, P-1
  splitters are chosen on that composite order (duplicate-heavy keys split
  by row id, which keeps stability), every rank range-partitions (K8 range
  variant), exchanges, and sorts locally with the stable radix sort. Rank r
  then holds the r-th slice of the global stable order.

On GPUs the exchange is fused with the partition gather: ``PeerExchange``
keeps every rank's receive buffers in symmetric memory, the P x P counts
go round once, and ``rl_push_rows`` reads each partitioned row from local
HBM and stores it straight into its destination's buffer through the peer
pointer (NVLink P2P), between two symmetric-memory barriers — the
all-to-all without a send buffer or a second pass (``RL_NO_P2P=1``, or a
group without symmetric memory, uses NCCL ``all_to_all_single``).

The device work is done through an ``Ops`` object: ``GpuOps`` calls the
sm_100a kernels; the CPU multi-process tests inject an oracle-backed
implementation to exercise this exchange protocol with the gloo backend
(there is one GPU in this environment).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

PARTITION_SEED = 0x5EED  # join partition hash seed (any fixed value; every rank must agree)


class GpuOps:
    """Device kernels for the distributed operators (librelab_b200.so)."""

    def hash_partition(self, keys: torch.Tensor, parts: int, seed: int):
        from . import engine

        return engine.hash_partition(keys, parts, seed)

    def range_partition(self, keys: torch.Tensor, gid_base: int, split_keys: torch.Tensor, split_gids: torch.Tensor,
                        descending: bool):
        from . import engine

        return engine.range_partition(keys, gid_base, split_keys, split_gids, descending)

    def take(self, col: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
        from . import engine

        rows = rows if rows.dtype == torch.int32 else rows.to(torch.int32)  # uint32 row-id bits
        out = torch.empty((rows.numel(),) + tuple(col.shape[1:]), dtype=col.dtype, device=col.device)
        width = col.element_size() * (col.shape[1] if col.dim() > 1 else 1)
        engine.gather_rows(rows, [engine.OutColumn(col.contiguous(), out, width, 0)])
        return out

    def local_join_pairs(self, lkeys: torch.Tensor, rkeys: torch.Tensor):
        """(left rows, right rows) of the local equi-join, int64, reference order."""
        from . import engine

        li, ri = engine.index_keys(lkeys), engine.index_keys(rkeys)
        al = engine.align(li, ri)
        m, total = engine.fetch_scalars(al.m_total)
        lr = torch.empty(total, dtype=torch.int32, device=lkeys.device)
        rr = torch.empty(total, dtype=torch.int32, device=lkeys.device)
        if total:
            engine.expand(al, m, li, ri, 0, total, (), lr, rr)
        return lr.to(torch.int64) & 0xFFFFFFFF, rr.to(torch.int64) & 0xFFFFFFFF

    def stable_order(self, keys: torch.Tensor, descending: bool) -> torch.Tensor:
        from . import engine

        perm = engine.sort_permutation([engine.SortAxis(keys, descending)], keys.numel(), keys.device)
        return perm.to(torch.int64) & 0xFFFFFFFF

    def push_exchange_many(self, items, group):
        """Partition gather + all-to-all in one kernel per exchange over peer
        memory (PeerExchange), for every exchange of a step at once: items are
        (slot, columns, partitioned rows, counts per destination, global row-id
        base); ONE all-gather of all count vectors (one host sync). Returns, per
        item, (received columns, their int64 global row ids, rows per source) —
        or None when this group has no symmetric memory."""
        if not items:
            return []
        from . import _capi as C

        dev = items[0][1][0].device
        if not _peer_exchange_ok(group, dev):
            return None
        # rl_push_rows limits: the same answer on every rank (same group, same
        # column lists), so this local check cannot split the group
        if _group_size(group) > C.RL_PUSH_MAX_PARTS or any(len(it[1]) > C.RL_PUSH_MAX_COLUMNS for it in items):
            return None
        exs = []
        for slot, cols, _, _, _ in items:
            key = (slot, id(group), dev.index, tuple((c.dtype, tuple(c.shape[1:])) for c in cols))
            if key not in _PEER:
                _PEER[key] = PeerExchange(group, dev, cols)
            exs.append(_PEER[key])
        return PeerExchange.exchange_many(exs, items, group)

    # fused forms (one launch for every column) used when an Ops object has them
    def local_join(self, lcols, lkey: int, rcols, rkey: int, lgids: torch.Tensor, rgids: torch.Tensor):
        """The local equi-join with every output column and both global row-id
        columns written by ONE expansion launch: the bucket join when it
        applies (payload and global ids carried with the rows), else the
        sort-based plan (rl_join_plan_build + rl_join_expand)."""
        from . import _capi as C
        from . import engine
        from .pipeline import join_out_columns

        plan = engine.plan_join(lcols[lkey], rcols[rkey],
                                [c for j, c in enumerate(lcols) if j != lkey] + [lgids],
                                [c for j, c in enumerate(rcols) if j != rkey] + [rgids])
        total = plan.total
        cols = join_out_columns(list(lcols), lkey, list(rcols), rkey, total)
        ids = [engine.OutColumn(lgids, torch.empty(total, dtype=torch.int64, device=lgids.device), 8, C.RL_SIDE_LEFT),
               engine.OutColumn(rgids, torch.empty(total, dtype=torch.int64, device=rgids.device), 8,
                                C.RL_SIDE_RIGHT)]
        if total:
            plan.expand(0, total, cols + ids)
        return [c.dst for c in cols], ids[0].dst, ids[1].dst

    def partition_take(self, kind: str, keys: torch.Tensor, cols: Sequence[torch.Tensor], **kw):
        """Partition + every column gathered into destination order in one
        gather launch (rl_hash_partition / rl_range_partition with columns)."""
        from . import engine

        outs = [torch.empty_like(c) for c in cols]
        oc = [engine.OutColumn(c.contiguous(), o, _row_bytes(c), 0) for c, o in zip(cols, outs)]
        if kind == "hash":
            rows, counts = engine.hash_partition(keys, kw["parts"], kw["seed"], columns=oc)
        else:
            rows, counts = engine.range_partition(keys, kw["gid_base"], kw["split_keys"], kw["split_gids"],
                                                  kw["descending"], columns=oc)
        return rows, counts, outs

    def sort_take(self, cols: Sequence[torch.Tensor], key_idx: int, descending: bool):
        """Stable sort by the int64 column key_idx: the sort kernel writes the
        sorted keys itself; every other column in one gather launch."""
        from . import engine

        keys = cols[key_idx]
        n = keys.numel()
        sk = torch.empty_like(keys)
        outs = [sk if j == key_idx else torch.empty_like(c) for j, c in enumerate(cols)]
        gather = [engine.OutColumn(c.contiguous(), outs[j], _row_bytes(c), 0) for j, c in enumerate(cols) if j != key_idx]
        if n:
            engine.sort_permutation([engine.SortAxis(keys, descending)], n, keys.device, sorted_keys_out=sk,
                                    gather=gather)
        return outs


class PeerExchange:
    """Receive buffers of one exchange slot in symmetric memory, and the
    fused partition-gather + all-to-all (rl_push_rows) into them. Received
    columns are views of the buffers, valid until this slot's next exchange."""

    def __init__(self, group, device, like: Sequence[torch.Tensor]):
        self.group, self.device = group, device
        self.p = _group_size(group)
        self.me = dist.get_rank(group)
        self.likes = [(c.dtype, tuple(c.shape[1:]), _row_bytes(c)) for c in like]
        self.cap = 0
        self._pending = None

    def _alloc(self, rows: int) -> bool:
        """Local half of a (re)allocation for `rows` received rows: the new
        symmetric buffer only (no collective). False on failure (e.g. OOM)."""
        import torch.distributed._symmetric_memory as sm

        cap = max(rows, self.cap + self.cap // 4, 1024)
        offs, total = [], 0
        for _, _, w in self.likes + [(None, None, 8)]:  # + the int64 global row ids
            offs.append(total)
            total += (cap * w + 255) // 256 * 256
        try:
            self._pending = (sm.empty(total, dtype=torch.uint8, device=self.device), offs, cap)
        except RuntimeError:
            self._pending = None
            return False
        return True

    def _commit(self) -> None:
        """Collective half: every rank allocated, so all of them rendezvous."""
        import torch.distributed._symmetric_memory as sm

        buf, offs, cap = self._pending
        self._pending = None
        grp = self.group if self.group is not None else dist.group.WORLD
        self.hdl = sm.rendezvous(buf, grp.group_name)
        self.buf = buf
        ptrs = list(self.hdl.buffer_ptrs)
        table = [[ptrs[d] + o for o in offs] for d in range(self.p)]  # user-space addresses < 2^63
        self.bases = torch.tensor(table, dtype=torch.int64).view(-1).to(self.device)
        self.offs, self.cap = offs, cap

    @staticmethod
    def exchange_many(exs, items, group):
        """One all-gather of every item's counts, then each item's push between
        two symmetric-memory barriers (see GpuOps.push_exchange_many)."""
        from . import _capi as C
        from . import engine

        p, me = exs[0].p, exs[0].me
        dev = exs[0].device
        mine = torch.cat([it[3].to(torch.int64).reshape(p) for it in items])
        gathered = torch.empty(p * mine.numel(), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gathered, mine, group=group)
        host = gathered.cpu().view(p, len(items), p)  # the step's one host sync; host[s][i][d]
        lib = C.load()
        # receive buffers that must grow: the same list on every rank (the same
        # counts matrix). Allocate locally, agree with a MIN all-reduce, and only
        # then rendezvous — a rank whose allocation failed takes the whole group
        # to NCCL instead of leaving its peers waiting in the rendezvous.
        grow = [(ex, int(host[:, i, :].sum(0).max())) for i, ex in enumerate(exs)]
        if not _grow_collectively([(ex, rows) for ex, rows in grow if rows > ex.cap], group, dev):
            _PEER[("ok", id(group), dev.index)] = False  # NCCL from now on, on every rank
            return None
        out_all = []
        for i, (ex, (_, cols, rows, counts, base)) in enumerate(zip(exs, items)):
            mat = host[:, i, :]  # mat[s][d]: rows s sends to d
            recv_counts = mat[:, me].tolist()
            total = sum(recv_counts)
            starts = torch.zeros(p + 1, dtype=torch.int64, device=dev)
            torch.cumsum(counts.to(torch.int64).reshape(p), 0, out=starts[1:])
            offs = torch.tensor([int(mat[:me, d].sum()) for d in range(p)], dtype=torch.int64).to(dev)
            arr, ncols = C.columns_array((c.contiguous().data_ptr(), 0, w, C.RL_SIDE_LEFT)
                                         for c, (_, _, w) in zip(cols, ex.likes))
            ex.hdl.barrier()  # every rank is done with its previous receive
            C.check(lib.rl_push_rows_gid(engine._ptr(rows), rows.numel(), p, engine._ptr(starts), arr, ncols,
                                         engine._ptr(ex.bases), engine._ptr(offs), int(base), engine.stream_handle()),
                    "rl_push_rows_gid")
            ex.hdl.barrier()  # every push into this rank has landed
            out = [ex.buf[o:o + total * w].view(dt).view((total,) + tail) for (dt, tail, w), o in zip(ex.likes, ex.offs)]
            gids = ex.buf[ex.offs[-1]:ex.offs[-1] + total * 8].view(torch.int64)
            out_all.append((out, gids, recv_counts))
        return out_all


_PEER: dict = {}


def _grow_collectively(grow, group, device) -> bool:
    """Grow receive buffers [(exchange, rows)] — the same list on every rank.
    Each rank allocates locally (``_alloc``), a MIN all-reduce agrees, and
    only if every rank succeeded do they all rendezvous (``_commit``).
    Returns False, on EVERY rank, if any rank failed to allocate."""
    if not grow:
        return True
    ok = all([ex._alloc(rows) for ex, rows in grow])
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if not bool(flag.item()):
        for ex, _ in grow:
            ex._pending = None
        return False
    for ex, _ in grow:
        ex._commit()
    return True


def _peer_exchange_ok(group, device) -> bool:
    if os.environ.get("RL_NO_P2P") or device.type != "cuda" or dist.get_backend(group) != "nccl":
        return False
    key = ("ok", id(group), device.index)
    if key not in _PEER:
        _PEER[key] = _probe_symmetric_memory(group, device)
    return _PEER[key]


def _probe_symmetric_memory(group, device) -> bool:
    """Whether EVERY rank of the group can use symmetric memory, decided
    collectively once: each rank tries a small buffer + rendezvous + barrier,
    then the ranks agree with a MIN all-reduce — no rank goes to the peer
    path while another falls back to NCCL (that would leave the two waiting
    on different collectives)."""
    ok = 1
    try:
        import torch.distributed._symmetric_memory as sm

        buf = sm.empty(4096, dtype=torch.uint8, device=device)
        grp = group if group is not None else dist.group.WORLD
        hdl = sm.rendezvous(buf, grp.group_name)
        hdl.barrier()
        torch.cuda.current_stream(device).synchronize()
        del hdl, buf
    except Exception:  # any failure on any rank: NCCL everywhere
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


def _row_bytes(c: torch.Tensor) -> int:
    return c.element_size() * (c.shape[1] if c.dim() > 1 else 1)


def _partition_take(ops, kind, keys, cols, **kw):
    if hasattr(ops, "partition_take"):
        return ops.partition_take(kind, keys, cols, **kw)
    if kind == "hash":
        rows, counts = ops.hash_partition(keys, kw["parts"], kw["seed"])
    else:
        rows, counts = ops.range_partition(keys, kw["gid_base"], kw["split_keys"], kw["split_gids"], kw["descending"])
    return rows, counts, [ops.take(c, rows) for c in cols]


def _sort_take(ops, cols, key_idx, descending):
    if hasattr(ops, "sort_take"):
        return ops.sort_take(cols, key_idx, descending)
    perm = ops.stable_order(cols[key_idx], descending)
    return [ops.take(c, perm) for c in cols]


def _global_ids(rows: torch.Tensor, recv_counts: list, bases: list) -> torch.Tensor:
    """int64 global row ids of received rows: the sender's base + its local
    row id (row ids travel as 4 bytes, not 8). One kernel on the GPU
    (rl_global_ids); torch ops on CPU tensors (the gloo tests)."""
    if rows.device.type == "cuda" and len(recv_counts) <= 64:
        import ctypes

        from . import _capi as C
        from . import engine

        p = len(recv_counts)
        out = torch.empty(rows.numel(), dtype=torch.int64, device=rows.device)
        rc = (ctypes.c_int64 * p)(*[int(c) for c in recv_counts])
        bs = (ctypes.c_int64 * p)(*[int(b) for b in bases])
        C.check(C.load().rl_global_ids(engine._ptr(rows), rows.numel(), p, rc, bs, engine._ptr(out),
                                       engine.stream_handle()), "rl_global_ids")
        return out
    r = rows.to(torch.int64) & 0xFFFFFFFF
    off = 0
    for c, b in zip(recv_counts, bases):  # P slices, one in-place add each
        if c and b:
            r[off:off + c] += b
        off += c
    return r


def _all_bases(base: int, device, group) -> list:
    t = torch.tensor([base], dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(_group_size(group))]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def _group_size(group) -> int:
    return dist.get_world_size(group)


def exchange(columns: Sequence[torch.Tensor], send_counts: torch.Tensor, group=None, with_counts: bool = False):
    """all-to-all-v of row-grouped columns. ``columns`` are grouped by
    destination rank (rank order), ``send_counts[d]`` rows for rank d. Returns
    the received columns, grouped by source rank, each group in source order
    (and the per-source row counts with ``with_counts``)."""
    p = _group_size(group)
    counts = send_counts.to(torch.int64).reshape(p)
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    send_l = counts.cpu().tolist()
    recv_l = recv_counts.cpu().tolist()
    out = []
    for col in columns:
        col = col.contiguous()
        dst = torch.empty((sum(recv_l),) + tuple(col.shape[1:]), dtype=col.dtype, device=col.device)
        dist.all_to_all_single(dst, col, output_split_sizes=recv_l, input_split_sizes=send_l, group=group)
        out.append(dst)
    return (out, recv_l) if with_counts else out


@dataclass
class JoinShard:
    """This rank's share of a distributed join's output."""

    columns: List[torch.Tensor]  # left columns (key = matched key), then right non-key columns
    left_gids: torch.Tensor  # int64 global row ids of the left rows
    right_gids: torch.Tensor  # int64 global row ids of the right rows
    total_matches: int  # all ranks


def distributed_join(left: Sequence[torch.Tensor], left_key: int, left_base: int, right: Sequence[torch.Tensor],
                     right_key: int, right_base: int, group=None, seed: int = PARTITION_SEED,
                     ops: Optional[object] = None) -> JoinShard:
    """Hash-partitioned equi-join of two row-sharded relations (see module doc)."""
    ops = ops or GpuOps()
    p = _group_size(group)
    dev = left[left_key].device

    def shuffle(cols, key_idx, base):
        bases = _all_bases(base, dev, group)
        rows, counts, moved = _partition_take(ops, "hash", cols[key_idx], list(cols), parts=p, seed=seed)
        recv, rc = exchange(moved + [rows], counts, group, with_counts=True)
        return recv[:-1], _global_ids(recv[-1], rc, bases)

    pushed = None
    if hasattr(ops, "push_exchange_many"):  # both sides' counts in one all-gather, global ids from the senders
        rl_, cl = ops.hash_partition(left[left_key], p, seed)
        rr_, cr = ops.hash_partition(right[right_key], p, seed)
        pushed = ops.push_exchange_many([("join_left", list(left), rl_, cl, left_base),
                                         ("join_right", list(right), rr_, cr, right_base)], group)
    if pushed is not None:
        (lcols, lgids, _), (rcols, rgids, _) = pushed
    else:
        lcols, lgids = shuffle(list(left), left_key, left_base)
        rcols, rgids = shuffle(list(right), right_key, right_base)
    if hasattr(ops, "local_join"):
        out, lg, rg = ops.local_join(lcols, left_key, rcols, right_key, lgids, rgids)
    else:
        lrows, rrows = ops.local_join_pairs(lcols[left_key], rcols[right_key])
        out = [ops.take(c, lrows) for c in lcols]
        out += [ops.take(c, rrows) for j, c in enumerate(rcols) if j != right_key]
        lg, rg = lgids[lrows], rgids[rrows]
    total = torch.tensor([lg.numel()], dtype=torch.int64, device=dev)
    dist.all_reduce(total, group=group)
    return JoinShard(out, lg, rg, int(total.item()))


def choose_splitters(keys: torch.Tensor, gid_base: int, descending: bool, group=None, per_rank: int = 256,
                     with_bases: bool = False):
    """Regular sampling of (key, global id); ONE all-gather of every rank's
    samples (and its row-id base); P-1 splitters on the composite order.
    Every rank computes the same splitters."""
    p = _group_size(group)
    n = keys.numel()
    m = min(per_rank, n)
    dev = keys.device
    idx = (torch.arange(per_rank, device=dev, dtype=torch.int64) * max(n, 1)) // max(m, 1)
    idx = idx.clamp_(max=max(n - 1, 0))
    head = torch.tensor([m, gid_base], dtype=torch.int64, device=dev)
    pack = torch.cat([head, keys[idx] if n else torch.zeros(per_rank, dtype=torch.int64, device=dev),
                      idx + gid_base])  # entries past m are ignored
    packs = torch.empty(p * pack.numel(), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(packs, pack, group=group)
    host = packs.cpu().view(p, -1)
    bases = [int(v) for v in host[:, 1].tolist()]
    ks = torch.cat([h[2:2 + int(h[0])] for h in host])
    gs = torch.cat([h[2 + per_rank:2 + per_rank + int(h[0])] for h in host])
    if ks.numel() == 0:
        e = torch.empty(0, dtype=torch.int64, device=dev)
        return (e, e, bases) if with_bases else (e, e)
    ordk = torch.bitwise_not(ks) if descending else ks
    # composite (key, gid) order: stable sort by gid then by key
    o = torch.argsort(gs, stable=True)
    o = o[torch.argsort(ordk[o], stable=True)]
    ks, gs = ks[o], gs[o]
    cnt = ks.numel()
    picks = [min(cnt - 1, (i * cnt) // p) for i in range(1, p)]
    both = torch.stack([ks[picks], gs[picks]])
    both = both.pin_memory().to(dev, non_blocking=True) if dev.type == "cuda" else both  # one small H2D
    sk, sg = both[0], both[1]
    return (sk, sg, bases) if with_bases else (sk, sg)


def choose_splitters_device(keys: torch.Tensor, gid_base: int, descending: bool, group=None, per_rank: int = 256):
    """choose_splitters without leaving the device: the gathered samples are
    ordered by (key, gid) and the P-1 splitters picked on the GPU (ranks
    with fewer rows contribute fewer samples; missing slots sort last)."""
    p = _group_size(group)
    n = keys.numel()
    dev = keys.device
    if dev.type == "cuda":  # two launches around the all-gather (rl_sample_keys, rl_pick_splitters)
        from . import _capi as C
        from . import engine

        lib = C.load()
        per = max(1, min(per_rank, C.RL_MAX_SPLIT_SAMPLES // p))
        keys = keys.contiguous()
        pack = torch.empty(3 * per, dtype=torch.int64, device=dev)
        C.check(lib.rl_sample_keys(engine._ptr(keys), n, per, int(gid_base), int(descending), engine._ptr(pack),
                                   engine.stream_handle()), "rl_sample_keys")
        allp = torch.empty(p * 3 * per, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(allp, pack, group=group)
        sk = torch.empty(max(p - 1, 0), dtype=torch.int64, device=dev)
        sg = torch.empty(max(p - 1, 0), dtype=torch.int64, device=dev)
        C.check(lib.rl_pick_splitters(engine._ptr(allp), p, per, int(descending), engine._ptr(sk), engine._ptr(sg),
                                      engine.stream_handle()), "rl_pick_splitters")
        return sk, sg
    m = min(per_rank, n)
    idx = (torch.arange(per_rank, device=dev, dtype=torch.int64) * max(n, 1)) // max(m, 1)
    idx = idx.clamp_(max=max(n - 1, 0))
    valid = torch.arange(per_rank, device=dev) < m
    k = keys[idx] if n else torch.zeros(per_rank, dtype=torch.int64, device=dev)
    ordk = torch.bitwise_not(k) if descending else k
    pack = torch.stack([ordk, idx + gid_base, valid.to(torch.int64)])  # [3, per_rank]
    allp = torch.empty((p * 3 * per_rank,), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allp, pack.reshape(-1), group=group)
    allp = allp.view(p, 3, per_rank).permute(1, 0, 2).reshape(3, -1)
    ok, gs, v = allp[0], allp[1], allp[2].bool()
    # composite (valid first, key, gid) order: stable sorts, least significant first
    o = torch.argsort(gs, stable=True)
    o = o[torch.argsort(ok[o], stable=True)]
    o = o[torch.argsort((~v[o]).to(torch.int8), stable=True)]
    cnt = v.sum()
    picks = (torch.arange(1, p, device=dev, dtype=torch.int64) * cnt) // p
    picks = torch.minimum(picks, (cnt - 1).clamp(min=0))
    sel = o[picks]
    sk = ok[sel]
    sk = torch.bitwise_not(sk) if descending else sk
    return sk, gs[sel]


@dataclass
class SortShard:
    columns: List[torch.Tensor]  # this rank's slice of the globally sorted relation
    gids: torch.Tensor  # their global row ids (the permutation slice)


def distributed_sort(cols: Sequence[torch.Tensor], key_idx: int, gid_base: int, descending: bool = False,
                     group=None, ops: Optional[object] = None) -> SortShard:
    """Range-partitioned stable ORDER BY on one int64 key (see module doc)."""
    ops = ops or GpuOps()
    keys = cols[key_idx]
    pushed = None
    if hasattr(ops, "push_exchange_many") and keys.device.type == "cuda" and _peer_exchange_ok(group, keys.device):
        # device-side splitters (no host sync); global row ids written by the senders
        split_k, split_g = choose_splitters_device(keys, gid_base, descending, group)
        rows, counts = ops.range_partition(keys, gid_base, split_k, split_g, descending)
        pushed = ops.push_exchange_many([("sort", list(cols), rows, counts, gid_base)], group)
    if pushed is not None:
        rcols, rgids, _ = pushed[0]
    else:
        split_k, split_g, bases = choose_splitters(keys, gid_base, descending, group, with_bases=True)
        rows, counts, moved = _partition_take(ops, "range", keys, list(cols), gid_base=gid_base, split_keys=split_k,
                                              split_gids=split_g, descending=descending)
        recv, rc = exchange(moved + [rows], counts, group, with_counts=True)
        rcols, rgids = recv[:-1], _global_ids(recv[-1], rc, bases)
    # arrival order = ascending global row id, so the stable local sort keeps the reference tie order
    out = _sort_take(ops, list(rcols) + [rgids], key_idx, descending)
    return SortShard(out[:-1], out[-1])
