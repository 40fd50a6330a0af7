"""bench.py's multi-GPU correctness gate (join_gate) on world size 2 (gloo,
CPU): each rank holds a row shard of both inputs and some of the join's
output rows (as after the hash-partitioned exchange); the per-key aggregates
and the observed sums are all-reduced. A correct split of the oracle's output
passes, a missing or altered row on one rank fails on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, corrupt, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import tensorpath_oracle as O

        n, dom = 20_000, 15_000
        rng = np.random.default_rng(3)
        lk, rk = rng.integers(0, dom, n), rng.integers(0, dom, n)
        pay = np.arange(n, dtype=np.int64)
        key, lp, rp = O.join_columns([lk, pay], 0, [rk, pay], 0)
        # inputs: contiguous row shards; outputs: the rows of keys hashed to this rank
        a, b = rank * n // world, (rank + 1) * n // world
        mine = (key % world) == rank
        ok, lq, rq = key[mine], lp[mine], rp[mine]
        if corrupt and rank == 1:
            rq = rq.copy()
            rq[5] += 1
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x))  # noqa: E731
        try:
            total = bench.join_gate([t(ok), t(lq), t(rq)], [t(lk[a:b]), t(pay[a:b])], [t(rk[a:b]), t(pay[a:b])],
                                    dom, world, torch.device("cpu"))
            out = ("ok", total, len(key))
        except SystemExit as e:
            out = ("rejected", str(e)[:80], len(key))
        got = [None] * world
        dist.all_gather_object(got, out)
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_join_gate_all_reduced_over_two_ranks(corrupt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, corrupt, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if corrupt:
        assert all(r[0] == "rejected" for r in res)
    else:
        assert all(r[0] == "ok" and r[1] == r[2] for r in res)
