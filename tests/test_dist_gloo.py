"""World-size-2 CPU tests (gloo) of the multi-GPU exchange protocol in
paper_2602_21237_b200/dist.py. The device kernels are replaced by an
oracle-backed Ops object (test infrastructure); partitioning, the
all-to-all-v exchange, global row-id bookkeeping, splitter choice and the
count all-reduce are the product code. Results are checked against the
single-process oracle on the unsharded relations."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tensorpath_oracle as O


class CpuOracleOps:
    """Same contract as dist.GpuOps, computed with the pinned numpy oracle."""

    def hash_partition(self, keys, parts, seed):
        k = keys.numpy().astype(np.int64)
        h = O.fmix64(k.view(np.uint64) ^ np.uint64(O.fmix64_scalar(seed)))
        dest = (h % np.uint64(parts)).astype(np.int64)
        rows = np.argsort(dest, kind="stable")
        return torch.from_numpy(rows.astype(np.int64)), torch.from_numpy(np.bincount(dest, minlength=parts))

    def range_partition(self, keys, gid_base, split_keys, split_gids, descending):
        k = keys.numpy().astype(np.int64)
        kk = np.invert(k) if descending else k
        sk = split_keys.numpy().astype(np.int64)
        sk = np.invert(sk) if descending else sk
        sg = split_gids.numpy()
        g = np.arange(len(k)) + gid_base
        dest = np.zeros(len(k), dtype=np.int64)
        for a, b in zip(sk, sg):
            dest += (a < kk) | ((a == kk) & (b < g))
        rows = np.argsort(dest, kind="stable")
        return torch.from_numpy(rows), torch.from_numpy(np.bincount(dest, minlength=len(sk) + 1))

    def take(self, col, rows):
        return col[rows.to(torch.int64)]

    def local_join_pairs(self, lkeys, rkeys):
        lr, rr = O.join_pairs(lkeys.numpy(), rkeys.numpy())
        return torch.from_numpy(lr), torch.from_numpy(rr)

    def stable_order(self, keys, descending):
        return torch.from_numpy(O.stable_axis_order(keys.numpy(), descending))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard(n, world, rank):
    base = (n * rank) // world
    return base, (n * (rank + 1)) // world


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_21237_b200 import dist as D

        ops = CpuOracleOps()
        rng = np.random.default_rng(case["seed"])
        if case["kind"] == "join":
            nl, nr, dom = case["nl"], case["nr"], case["dom"]
            lk = rng.integers(-dom, dom, nl).astype(np.int64)
            rk = rng.integers(-dom, dom, nr).astype(np.int64)
            lp = rng.integers(0, 256, (nl, 3), dtype=np.uint8)
            rp = np.arange(nr, dtype=np.int64) * 7
            la, lb = _shard(nl, world, rank)
            ra, rb = _shard(nr, world, rank)
            res = D.distributed_join([torch.from_numpy(lk[la:lb]), torch.from_numpy(lp[la:lb])], 0, la,
                                     [torch.from_numpy(rp[ra:rb]), torch.from_numpy(rk[ra:rb])], 1, ra,
                                     ops=ops)
            out = {"lg": res.left_gids.numpy(), "rg": res.right_gids.numpy(), "total": res.total_matches,
                   "cols": [c.numpy() for c in res.columns]}
        elif case["kind"] == "splitters":
            n = case["n"]
            keys = rng.integers(-case["dom"], case["dom"], n).astype(np.int64)
            a, b = _shard(n, world, rank)
            kt = torch.from_numpy(keys[a:b])
            hk, hg = D.choose_splitters(kt, a, case["desc"])
            dk, dg = D.choose_splitters_device(kt, a, case["desc"])
            out = {"host": (hk.numpy(), hg.numpy()), "dev": (dk.numpy(), dg.numpy())}
        elif case["kind"] == "grow":
            # receive-buffer growth: rank `fail` cannot allocate; every rank must
            # get False (NCCL fallback) and nobody may enter the rendezvous
            class FakeExchange:
                cap = 0
                _pending = None
                committed = False

                def _alloc(self, rows):
                    if rank == case["fail"]:
                        return False
                    self._pending = rows
                    return True

                def _commit(self):
                    self.committed = True
                    self.cap = self._pending

            exs = [FakeExchange(), FakeExchange()]
            ok = D._grow_collectively([(exs[0], 100), (exs[1], 200)], None, torch.device("cpu"))
            out = {"ok": ok, "committed": [e.committed for e in exs], "caps": [e.cap for e in exs],
                   "pending": [e._pending for e in exs]}
        else:
            n = case["n"]
            keys = rng.integers(-case["dom"], case["dom"], n).astype(np.int64)
            pay = rng.integers(0, 256, (n, 2), dtype=np.uint8)
            a, b = _shard(n, world, rank)
            res = D.distributed_sort([torch.from_numpy(keys[a:b]), torch.from_numpy(pay[a:b])], 0, a,
                                     descending=case["desc"], ops=ops)
            out = {"gids": res.gids.numpy(), "cols": [c.numpy() for c in res.columns]}
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_join_matches_single_process(world):
    case = {"kind": "join", "seed": 5, "nl": 3000, "nr": 2500, "dom": 300}
    parts = _run(case, world)
    rng = np.random.default_rng(5)
    lk = rng.integers(-300, 300, 3000).astype(np.int64)
    rk = rng.integers(-300, 300, 2500).astype(np.int64)
    lp = rng.integers(0, 256, (3000, 3), dtype=np.uint8)
    rp = np.arange(2500, dtype=np.int64) * 7
    wl, wr = O.join_pairs(lk, rk)
    assert all(p["total"] == len(wl) for p in parts)
    lg = np.concatenate([p["lg"] for p in parts])
    rg = np.concatenate([p["rg"] for p in parts])
    # the north-star canonicalisation: identical multiset of (r_idx, s_idx)
    assert O.canonical_pairs_sha256(lg, rg) == O.canonical_pairs_sha256(wl, wr)
    # every shard's rows are the reference rows of its pairs, in (key, l, r) order per key
    for p in parts:
        key, lpay, rpay = p["cols"]
        assert (key == lk[p["lg"]]).all() and (lpay == lp[p["lg"]]).all() and (rpay == rp[p["rg"]]).all()
        order = np.lexsort((p["rg"], p["lg"], key))
        assert (order == np.arange(len(order))).all()


@pytest.mark.parametrize("desc", [False, True])
def test_distributed_sort_is_the_global_stable_order(desc):
    case = {"kind": "sort", "seed": 9, "n": 5000, "dom": 40, "desc": desc}
    parts = _run(case, 2)
    rng = np.random.default_rng(9)
    keys = rng.integers(-40, 40, 5000).astype(np.int64)
    pay = rng.integers(0, 256, (5000, 2), dtype=np.uint8)
    want = O.stable_axis_order(keys, desc)
    gids = np.concatenate([p["gids"] for p in parts])
    assert (gids == want).all()
    assert (np.concatenate([p["cols"][0] for p in parts]) == keys[want]).all()
    assert (np.concatenate([p["cols"][1] for p in parts]) == pay[want]).all()
    assert min(len(p["gids"]) for p in parts) > 1000  # splitters balance heavy duplicates


def test_exchange_counts_and_order_two_ranks():
    case = {"kind": "join", "seed": 1, "nl": 1, "nr": 0, "dom": 3}
    parts = _run(case, 2)
    assert all(p["total"] == 0 for p in parts)


@pytest.mark.parametrize("desc", [False, True])
def test_device_splitters_match_host_splitters(desc):
    """choose_splitters_device (no host round trip) picks the same (key, gid)
    splitters as the host version, duplicates included."""
    parts = _run({"kind": "splitters", "seed": 13, "n": 3001, "dom": 50, "desc": desc}, 2)
    for p in parts:
        assert (p["host"][0] == p["dev"][0]).all() and (p["host"][1] == p["dev"][1]).all()


@pytest.mark.parametrize("fail", [-1, 0, 1])
def test_peer_buffer_growth_is_agreed_by_every_rank(fail):
    """a rank that cannot allocate its symmetric receive buffer must
    take the WHOLE group to the NCCL path (a MIN all-reduce before any
    rendezvous), not fall back alone while its peers wait in the rendezvous."""
    parts = _run({"kind": "grow", "seed": 0, "fail": fail}, 2)
    for p in parts:
        if fail < 0:
            assert p["ok"] and p["committed"] == [True, True] and p["caps"] == [100, 200]
        else:
            assert not p["ok"] and p["committed"] == [False, False] and p["pending"] == [None, None]
