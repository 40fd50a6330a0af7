"""The distributed operators on the real device kernels (GpuOps) in a
one-rank NCCL group: partition, exchange (trivial), local join / sort."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import tensorpath_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    if dist.is_initialized():
        yield
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("plan", ["sort", "bucket"])
def test_distributed_join_on_device(nccl_world1, plan, monkeypatch):
    """The local join after the exchange through either plan: the bucket join
    (forced at this size; left payload + global id too wide to carry, right
    payload + global id carried) or the sort-based plan."""
    from paper_2602_21237_b200 import dist as D

    monkeypatch.setenv("RL_FORCE_BJOIN" if plan == "bucket" else "RL_NO_BJOIN", "1")

    rng = np.random.default_rng(3)
    lk = rng.integers(0, 5000, 40_000).astype(np.int64)
    rk = rng.integers(0, 5000, 30_000).astype(np.int64)
    lp = rng.integers(0, 256, (40_000, 16), dtype=np.uint8)
    rp = np.arange(30_000, dtype=np.int64)
    res = D.distributed_join([torch.from_numpy(lk).cuda(), torch.from_numpy(lp).cuda()], 0, 0,
                             [torch.from_numpy(rk).cuda(), torch.from_numpy(rp).cuda()], 0, 0)
    wl, wr = O.join_pairs(lk, rk)
    assert res.total_matches == len(wl)
    assert (res.left_gids.cpu().numpy() == wl).all() and (res.right_gids.cpu().numpy() == wr).all()
    assert (res.columns[1].cpu().numpy() == lp[wl]).all()
    assert (res.columns[2].cpu().numpy() == rp[wr]).all()


def test_distributed_sort_on_device(nccl_world1):
    from paper_2602_21237_b200 import dist as D

    rng = np.random.default_rng(4)
    keys = rng.integers(-(2**40), 2**40, 50_000).astype(np.int64)
    keys[::3] = 7
    res = D.distributed_sort([torch.from_numpy(keys).cuda()], 0, 0, descending=True)
    want = O.stable_axis_order(keys, True)
    assert (res.gids.cpu().numpy() == want).all()
    assert (res.columns[0].cpu().numpy() == keys[want]).all()


@pytest.mark.parametrize("gid", [False, True])
def test_push_rows_emulated_ranks(gid):
    """rl_push_rows for P logical ranks on one GPU (each rank's receive
    buffers are separate allocations; ranks push one after another, none
    waits on another): every destination receives source blocks in rank
    order, each in stable partition order, with the local row ids — the
    all-to-all-v contract. rl_push_rows_gid
    delivers int64 global row ids (the sender's base + its local row id)."""
    import ctypes

    from paper_2602_21237_b200 import _capi as C
    from paper_2602_21237_b200 import engine

    lib = C.load()
    P = 3
    rng = np.random.default_rng(21)
    sizes = [40_000, 0, 65_537]
    keys = [rng.integers(-10**6, 10**6, n).astype(np.int64) for n in sizes]
    pays = [rng.integers(0, 256, (n, 12), dtype=np.uint8) for n in sizes]
    parts = []
    for k in keys:
        rows, counts = engine.hash_partition(torch.from_numpy(k).cuda(), P, 77)
        parts.append((rows, counts.cpu().numpy()))
    mat = np.stack([c for _, c in parts])  # mat[s][d]
    recv = mat.sum(0)
    gbase = [10**11, 7, 2**40]  # the senders' first global row ids
    bufs = [(torch.empty(max(r, 1), dtype=torch.int64, device="cuda"),
             torch.empty((max(r, 1), 12), dtype=torch.uint8, device="cuda"),
             torch.empty(max(r, 1), dtype=torch.int64 if gid else torch.int32, device="cuda")) for r in recv]
    table = torch.tensor([[b[0].data_ptr(), b[1].data_ptr(), b[2].data_ptr()] for b in bufs],
                         dtype=torch.int64).view(-1).cuda()
    for s in range(P):
        rows, counts = parts[s]
        kd, pd = torch.from_numpy(keys[s]).cuda(), torch.from_numpy(pays[s]).cuda()
        starts = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int64).cuda()
        offs = torch.tensor([int(mat[:s, d].sum()) for d in range(P)], dtype=torch.int64).cuda()
        arr, ncols = C.columns_array([(kd.data_ptr(), 0, 8, C.RL_SIDE_LEFT), (pd.data_ptr(), 0, 12, C.RL_SIDE_LEFT)])
        if gid:
            C.check(lib.rl_push_rows_gid(ctypes.c_void_p(rows.data_ptr()), rows.numel(), P,
                                         ctypes.c_void_p(starts.data_ptr()), arr, ncols,
                                         ctypes.c_void_p(table.data_ptr()), ctypes.c_void_p(offs.data_ptr()),
                                         gbase[s], engine.stream_handle()), "rl_push_rows_gid")
        else:
            C.check(lib.rl_push_rows(ctypes.c_void_p(rows.data_ptr()), rows.numel(), P,
                                     ctypes.c_void_p(starts.data_ptr()), arr, ncols, ctypes.c_void_p(table.data_ptr()),
                                     ctypes.c_void_p(offs.data_ptr()), engine.stream_handle()), "rl_push_rows")
    torch.cuda.synchronize()
    for d in range(P):
        want_rows = [np.flatnonzero(O.fmix64(keys[s].view(np.uint64) ^ np.uint64(O.fmix64_scalar(77)))
                                    % np.uint64(P) == d) for s in range(P)]
        wk = np.concatenate([keys[s][r] for s, r in enumerate(want_rows)])
        wp = np.concatenate([pays[s][r] for s, r in enumerate(want_rows)])
        wr = np.concatenate(want_rows)
        n = int(recv[d])
        assert (bufs[d][0][:n].cpu().numpy() == wk).all()
        assert (bufs[d][1][:n].cpu().numpy() == wp).all()
        if gid:
            wg = np.concatenate([r.astype(np.int64) + gbase[s] for s, r in enumerate(want_rows)])
            assert (bufs[d][2][:n].cpu().numpy() == wg).all()
        else:
            assert (bufs[d][2][:n].cpu().numpy().view(np.uint32) == wr).all()


def test_distributed_ops_take_the_peer_push(nccl_world1, monkeypatch):
    """One-rank NCCL group: the distributed sort and join go through
    PeerExchange (symmetric memory) and agree with the NCCL all-to-all path."""
    from paper_2602_21237_b200 import dist as D

    rng = np.random.default_rng(5)
    keys = rng.integers(-(2**40), 2**40, 80_000).astype(np.int64)
    pay = rng.integers(0, 256, (80_000, 4), dtype=np.uint8)
    kd, pd = torch.from_numpy(keys).cuda(), torch.from_numpy(pay).cuda()
    a = D.distributed_sort([kd, pd], 0, 0)
    monkeypatch.setenv("RL_NO_P2P", "1")
    b = D.distributed_sort([kd, pd], 0, 0)
    monkeypatch.delenv("RL_NO_P2P")
    assert torch.equal(a.gids, b.gids) and torch.equal(a.columns[1], b.columns[1])
    assert (a.gids.cpu().numpy() == O.stable_axis_order(keys, False)).all()
    lk = rng.integers(0, 5000, 30_000).astype(np.int64)
    rk = rng.integers(0, 5000, 20_000).astype(np.int64)
    j = D.distributed_join([torch.from_numpy(lk).cuda()], 0, 0, [torch.from_numpy(rk).cuda()], 0, 0)
    wl, wr = O.join_pairs(lk, rk)
    assert (j.left_gids.cpu().numpy() == wl).all() and (j.right_gids.cpu().numpy() == wr).all()
    used = [k for k in D._PEER if k[0] in ("sort", "join_left", "join_right")]
    assert used, "the peer-memory exchange was not used"


@pytest.mark.parametrize("descending", [False, True])
def test_splitter_and_gid_kernels_emulated_ranks(descending):
    """rl_sample_keys / rl_pick_splitters / rl_global_ids for five emulated
    ranks (one with fewer rows than samples, duplicate-heavy keys) against a
    numpy restatement: samples at i * n // m, splitters at ranks j * cnt // P
    of the (real first, key, global id) order, gid = sender base + local row."""
    import ctypes

    from paper_2602_21237_b200 import _capi as C
    from paper_2602_21237_b200 import engine

    lib = C.load()
    rng = np.random.default_rng(31 + descending)
    sizes = [5000, 3000, 100, 7000, 4000]
    per = 256
    p = len(sizes)
    bases = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    packs = []
    for n, b in zip(sizes, bases):
        keys = rng.integers(-50, 50, n).astype(np.int64)  # heavy duplicates: ties split by global id
        kd = torch.from_numpy(keys).cuda()
        pack = torch.empty(3 * per, dtype=torch.int64, device="cuda")
        C.check(lib.rl_sample_keys(engine._ptr(kd), n, per, int(b), int(descending), engine._ptr(pack),
                                   engine.stream_handle()), "rl_sample_keys")
        m = min(per, n)
        idx = np.minimum(np.arange(per) * max(n, 1) // max(m, 1), n - 1)
        want = np.stack([~keys[idx] if descending else keys[idx], idx + b, (np.arange(per) < m).astype(np.int64)])
        assert (pack.cpu().numpy().reshape(3, per) == want).all()
        packs.append(want)
    allp = torch.from_numpy(np.concatenate([q.reshape(-1) for q in packs])).cuda()
    sk = torch.empty(p - 1, dtype=torch.int64, device="cuda")
    sg = torch.empty(p - 1, dtype=torch.int64, device="cuda")
    C.check(lib.rl_pick_splitters(engine._ptr(allp), p, per, int(descending), engine._ptr(sk), engine._ptr(sg),
                                  engine.stream_handle()), "rl_pick_splitters")
    k = np.concatenate([q[0] for q in packs])
    g = np.concatenate([q[1] for q in packs])
    v = np.concatenate([q[2] for q in packs])
    order = np.lexsort((g, k, 1 - v))  # real samples first, then key, then global id
    cnt = int(v.sum())
    picks = np.minimum(np.arange(1, p) * cnt // p, cnt - 1)
    want_k = k[order[picks]]
    assert (sk.cpu().numpy() == (~want_k if descending else want_k)).all()
    assert (sg.cpu().numpy() == g[order[picks]]).all()

    recv = [300, 0, 17, 1200, 5]
    rows = rng.integers(0, 2**32, sum(recv), dtype=np.uint64).astype(np.uint32)
    rd = torch.from_numpy(rows.view(np.int32)).cuda()
    out = torch.empty(len(rows), dtype=torch.int64, device="cuda")
    rb = [10**12, 5, 0, 2**40 + 3, 77]
    C.check(lib.rl_global_ids(engine._ptr(rd), len(rows), p, (ctypes.c_int64 * p)(*recv), (ctypes.c_int64 * p)(*rb),
                              engine._ptr(out), engine.stream_handle()), "rl_global_ids")
    want_g = rows.astype(np.int64) + np.repeat(np.array(rb, dtype=np.int64), recv)
    assert (out.cpu().numpy() == want_g).all()
