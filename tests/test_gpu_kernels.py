"""Kernel-level GPU parity through the C ABI (engine.py → librelab_b200.so):
sizes that straddle tile boundaries, every key shape the onesweep passes
see, and the partition / gather / widen primitives."""

import numpy as np
import pytest
import torch

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import engine

pytestmark = pytest.mark.gpu

SIZES = [2, 3, 5, 16, 17, 31, 33, 40, 80, 255, 333, 511, 700, 3071, 3072, 3073, 3583, 3584, 3585, 6143, 6145,
         7000, 7167, 7169, 50_000]


def keys_for(n, mode, seed):
    rng = np.random.default_rng(seed)
    if mode == "neg":
        return rng.integers(-8, 8, n).astype(np.int64)
    if mode == "wide":
        return rng.integers(-(2**62), 2**62, n).astype(np.int64)
    if mode == "const":
        return np.full(n, -5, dtype=np.int64)
    if mode == "extreme":
        return rng.choice(np.array([-(2**63), 2**63 - 1, 0, -1], dtype=np.int64), n)
    return rng.integers(0, 4, n).astype(np.int64)


def u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32).astype(np.int64)


@pytest.mark.parametrize("mode", ["neg", "wide", "small", "const", "extreme"])
def test_sort_axis_sizes_and_shapes(mode):
    for n in SIZES:
        keys = keys_for(n, mode, n)
        kd = torch.from_numpy(keys).cuda()
        for desc in (False, True):
            sk = torch.empty(n, dtype=torch.int64, device="cuda")
            perm = engine.sort_permutation([engine.SortAxis(kd, desc)], n, kd.device, sorted_keys_out=sk)
            want = O.stable_axis_order(keys, desc)
            got = u32(perm)
            assert (got == want).all(), (n, mode, desc)
            assert (sk.cpu().numpy() == keys[want]).all(), (n, mode, desc)


def test_sort_refinement_with_perm_in_and_bytes_words():
    rng = np.random.default_rng(4)
    for n in (1, 2, 17, 3073, 9000):
        a = rng.integers(-3, 3, n).astype(np.int64)
        w = rng.integers(0, 3, (n, 11), dtype=np.uint8)
        dev = [engine.SortAxis(torch.from_numpy(a).cuda(), True), engine.SortAxis(torch.from_numpy(w).cuda(), False)]
        perm = engine.sort_permutation(dev, n, "cuda")
        assert (u32(perm) == O.sort_permutation([a, w], [True, False])).all(), n


def test_run_bounds_and_empty_index():
    for n in (0, 1, 2, 4095, 4096, 4097, 20_000):
        keys = np.random.default_rng(n).integers(-5, 5, n).astype(np.int64)
        idx = engine.index_keys(torch.from_numpy(keys).cuda())
        kv, off, pos = O.to_tensor_arrays(keys)
        d = engine.fetch_scalars(idx.d)[0]
        assert d == len(kv)
        assert idx.key_values[:d].cpu().tolist() == kv.tolist()
        assert u32(idx.offsets[: d + 1]).tolist() == off.tolist()
        assert u32(idx.positions).tolist() == pos.tolist()


def test_align_matches_oracle_with_gaps():
    rng = np.random.default_rng(12)
    for nl, nr in ((1, 1), (5000, 1), (1, 5000), (30_000, 20_000), (0, 10)):
        lk = rng.integers(0, 4000, nl).astype(np.int64)
        rk = rng.integers(2000, 6000, nr).astype(np.int64)
        li, ri = engine.index_keys(torch.from_numpy(lk).cuda()), engine.index_keys(torch.from_numpy(rk).cuda())
        al = engine.align(li, ri)
        m, total = engine.fetch_scalars(al.m_total)
        a = O.to_tensor_arrays(lk)
        b = O.to_tensor_arrays(rk)
        mk, ls, lc, rs, rc = O.align_arrays(a[0], a[1], b[0], b[1])
        assert m == len(mk) and total == int((lc * rc).sum())
        if m:
            assert al.matched_keys[:m].cpu().tolist() == mk.tolist()
            assert u32(al.left_counts[:m]).tolist() == lc.tolist()
            assert u32(al.right_starts[:m]).tolist() == rs.tolist()


@pytest.mark.parametrize("prepass", ["0", "1"])
def test_align_window_paths(monkeypatch, prepass):
    """key_axis.cu's alignment with the window pre-pass forced off / on, over
    multi-tile left axes (2048 keys per tile) whose right windows are narrower
    than, about equal to and wider than the 2560 staged keys (the per-key global
    search), and a right side that ends inside the left range."""
    monkeypatch.setenv("RL_ALIGN_PREPASS", prepass)
    rng = np.random.default_rng(21)
    cases = [
        (rng.choice(10**6, 40_000, replace=False), rng.choice(10**6, 40_000, replace=False)),  # balanced
        (rng.choice(10**5, 9_000, replace=False), np.arange(0, 10**5, 2)),  # right 5x denser: wide windows
        (np.arange(0, 60_000, 3), rng.choice(60_000, 700, replace=False)),  # sparse right
        (np.arange(50_000), np.arange(30_000, 31_000)),  # right ends inside the left range
        (np.arange(10_000), np.arange(20_000, 25_000)),  # disjoint
    ]
    for lk, rk in cases:
        lk = np.repeat(np.asarray(lk, np.int64), 1 + (np.arange(len(lk)) % 3))  # multiplicities 1-3
        rk = np.asarray(rk, np.int64)
        li, ri = engine.index_keys(torch.from_numpy(lk).cuda()), engine.index_keys(torch.from_numpy(rk).cuda())
        al = engine.align(li, ri)
        m, total = engine.fetch_scalars(al.m_total)
        a, b = O.to_tensor_arrays(lk), O.to_tensor_arrays(rk)
        mk, ls, lc, rs, rc = O.align_arrays(a[0], a[1], b[0], b[1])
        assert m == len(mk) and total == int((lc * rc).sum()), (prepass, len(lk), len(rk))
        if m:
            assert al.matched_keys[:m].cpu().tolist() == mk.tolist()
            assert u32(al.left_counts[:m]).tolist() == lc.tolist()
            assert u32(al.right_starts[:m]).tolist() == rs.tolist()


def test_expand_chunks_equal_full():
    rng = np.random.default_rng(13)
    lk = rng.integers(0, 300, 20_000).astype(np.int64)
    rk = rng.integers(0, 300, 10_000).astype(np.int64)
    li, ri = engine.index_keys(torch.from_numpy(lk).cuda()), engine.index_keys(torch.from_numpy(rk).cuda())
    al = engine.align(li, ri)
    m, total = engine.fetch_scalars(al.m_total)
    wl, wr = O.join_pairs(lk, rk)
    step = 1_234_567
    for a in range(0, total, step):
        b = min(a + step, total)
        lr = torch.empty(b - a, dtype=torch.int32, device="cuda")
        rr = torch.empty(b - a, dtype=torch.int32, device="cuda")
        engine.expand(al, m, li, ri, a, b, (), lr, rr)
        assert (u32(lr) == wl[a:b]).all() and (u32(rr) == wr[a:b]).all()


def test_hash_partition_is_stable_and_matches_hash_i64(golden):
    _, arr = golden
    keys = np.concatenate([arr["hash_keys"], np.random.default_rng(2).integers(-1000, 1000, 20_000)]).astype(np.int64)
    n = len(keys)
    payload = np.arange(n, dtype=np.int64) * 3
    for parts in (1, 2, 3, 8):
        kd = torch.from_numpy(keys).cuda()
        pd = torch.from_numpy(payload).cuda()
        out_pay = torch.empty(n, dtype=torch.int64, device="cuda")
        rows, counts = engine.hash_partition(kd, parts, 7, [engine.OutColumn(pd, out_pay, 8, 0)])
        h = O.fmix64(keys.view(np.uint64) ^ np.uint64(O.fmix64_scalar(7)))
        dest = (h % np.uint64(parts)).astype(np.int64)
        want_rows = np.argsort(dest, kind="stable")
        assert (u32(rows) == want_rows).all(), parts
        assert counts.cpu().tolist() == np.bincount(dest, minlength=parts).tolist()
        assert (out_pay.cpu().numpy() == payload[want_rows]).all()
    # seed 7 hash values are the reference's hash_i64 (hashing.py:54-61)
    assert (O.fmix64(arr["hash_keys"].view(np.uint64) ^ np.uint64(O.fmix64_scalar(7))) == arr["hash_seed7"]).all()


def test_gather_and_widen_widths():
    rng = np.random.default_rng(5)
    n, m = 1000, 4321
    rows = rng.integers(0, n, m).astype(np.uint32)
    rows_d = torch.from_numpy(rows.view(np.int32)).cuda()
    for w in (0, 1, 3, 4, 8, 12, 16, 24, 92):
        src = rng.integers(0, 256, (n, w), dtype=np.uint8)
        dst = torch.empty((m, w), dtype=torch.uint8, device="cuda")
        engine.gather_rows(rows_d, [engine.OutColumn(torch.from_numpy(src).cuda(), dst, w, 0)])
        assert (dst.cpu().numpy() == src[rows]).all(), w
    wide = engine.widen(rows_d)
    assert (wide.cpu().numpy() == rows.astype(np.int64)).all()


def test_range_partition_matches_composite_order():
    rng = np.random.default_rng(21)
    for desc in (False, True):
        n = 20_000
        keys = rng.integers(-50, 50, n).astype(np.int64)
        base = 1000
        split_k = np.array([-10, 0, 0, 30], dtype=np.int64)
        split_g = np.array([5000, 1500, 12000, 4000], dtype=np.int64)
        if desc:
            split_k = split_k[::-1].copy()
        rows, counts = engine.range_partition(torch.from_numpy(keys).cuda(), base, torch.from_numpy(split_k),
                                              torch.from_numpy(split_g), desc)
        kk = np.invert(keys) if desc else keys
        sk = np.invert(split_k) if desc else split_k
        g = np.arange(n) + base
        dest = np.zeros(n, dtype=np.int64)
        for a, b in zip(sk, split_g):
            dest += (a < kk) | ((a == kk) & (b < g))
        assert (u32(rows) == np.argsort(dest, kind="stable")).all()
        assert counts.cpu().tolist() == np.bincount(dest, minlength=5).tolist()


def test_fused_final_pass_gather_equals_take():
    rng = np.random.default_rng(31)
    for n in (1, 5, 3073, 40_000):
        keys = rng.integers(-100, 100, n).astype(np.int64)
        cols = [rng.integers(0, 256, (n, w), dtype=np.uint8) for w in (1, 4, 12, 16)]
        cols.append(np.arange(n, dtype=np.int64) * 3)
        gathers = []
        for c in cols:
            src = torch.from_numpy(c).cuda()
            dst = torch.empty_like(src)
            gathers.append(engine.OutColumn(src, dst, c.itemsize * (c.shape[1] if c.ndim > 1 else 1), 0))
        for desc in (False, True):
            perm = engine.sort_permutation([engine.SortAxis(torch.from_numpy(keys).cuda(), desc)], n, "cuda",
                                           gather=gathers, fuse_gather=(n % 2 == 1))
            want = O.stable_axis_order(keys, desc)
            assert (u32(perm) == want).all()
            for c, g in zip(cols, gathers):
                assert (g.dst.cpu().numpy() == c[want]).all(), (n, c.shape)
    # constant keys: no active digit, the copy-through path gathers too
    keys = np.full(1000, 3, dtype=np.int64)
    src = torch.arange(1000, dtype=torch.int64, device="cuda")
    dst = torch.empty_like(src)
    engine.sort_permutation([engine.SortAxis(torch.from_numpy(keys).cuda())], 1000, "cuda",
                            gather=[engine.OutColumn(src, dst, 8, 0)], fuse_gather=True)
    assert (dst.cpu().numpy() == np.arange(1000)).all()


def test_sort_graph_fallback_node_follows_each_replay():
    """Scatter-path SortGraph: the LSD fallback sits in a conditional node that
    the local phase arms per replay. Uniform keys, then one sub-bucket above
    the on-chip cap (the fallback runs), then keys with constant top bits
    (the pre-check falls back), then uniform again: every replay is exact."""
    n = 5_000_000
    rng = np.random.default_rng(77)
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    g = engine.SortGraph(keys)
    uniform = lambda: rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64, endpoint=True)  # noqa: E731
    hot = uniform()
    idx = rng.choice(n, 4000, replace=False)
    hot[idx] = (np.int64(0x1234) << 48) | rng.integers(0, 1 << 48, 4000, dtype=np.int64)
    narrow = rng.integers(0, 1 << 40, n, dtype=np.int64)
    for k in (uniform(), hot, narrow, uniform()):
        keys.copy_(torch.from_numpy(k))
        g.replay()
        want = O.stable_axis_order(k, False)
        assert (u32(g.perm) == want).all()
        assert (g.sorted_keys.cpu().numpy() == k[want]).all()


def test_sort_graph_replays_current_inputs():
    """engine.SortGraph: a captured sort + gather re-sorts whatever the bound
    input buffers hold at replay time (hybrid-sized and LSD-sized inputs)."""
    for n in (300_000, 5000):
        rng = np.random.default_rng(n)
        keys = torch.empty(n, dtype=torch.int64, device="cuda")
        pay = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
        out = torch.empty_like(pay)
        g = engine.SortGraph(keys, gather=[engine.OutColumn(pay, out, 4, 0)])
        for seed in (1, 2):
            k = rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64, endpoint=True)
            p = rng.integers(0, 256, (n, 4), dtype=np.uint8)
            keys.copy_(torch.from_numpy(k))
            pay.copy_(torch.from_numpy(p))
            g.replay()
            want = O.stable_axis_order(k, False)
            assert (u32(g.perm) == want).all()
            assert (g.sorted_keys.cpu().numpy() == k[want]).all()
            assert (out.cpu().numpy() == p[want]).all()
