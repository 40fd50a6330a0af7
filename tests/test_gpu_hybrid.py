"""The wide-key hybrid sort (radix_sort.cu: the rows reach their 65536
sub-buckets — top 16 key bits — by two top-digit onesweep passes or by the
scatter path's chunk counts + two non-stable counting passes; an on-chip local sort of
every sub-bucket; LSD fallback on skew) against the reference's stable
argsort (tensorpath.py:62-75, 206-216 via the oracle).

Every case is checked for the permutation (stable tie order) and the sorted
key values; the shapes are chosen to reach each branch of the local phase
and every fallback point. Each test runs through both ways into the
sub-buckets: RL_SCATTER_MIN_ROWS
lowers the scatter threshold to the hybrid's, RL_NO_SCATTER forces the passes."""

import numpy as np
import pytest
import torch

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import engine

pytestmark = pytest.mark.gpu

LOCAL_CAP = 2560  # kLocalCap in radix_sort.cu
I64_MIN, I64_MAX = -(2**63), 2**63 - 1


@pytest.fixture(autouse=True, params=["scatter", "passes"])
def into_subbuckets(request, monkeypatch):
    if request.param == "passes":
        monkeypatch.setenv("RL_NO_SCATTER", "1")
    else:
        monkeypatch.setenv("RL_SCATTER_MIN_ROWS", str(1 << 18))
    return request.param


def check_sort(keys: np.ndarray, desc: bool = False):
    n = len(keys)
    kd = torch.from_numpy(keys).cuda()
    sk = torch.empty(n, dtype=torch.int64, device="cuda")
    perm = engine.sort_permutation([engine.SortAxis(kd, desc)], n, kd.device, sorted_keys_out=sk)
    got = perm.cpu().numpy().view(np.uint32).astype(np.int64)
    want = O.stable_axis_order(keys, desc)
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (n, desc, bad[:5], got[bad[:5]], want[bad[:5]])
    assert (sk.cpu().numpy() == keys[want]).all()


def full_range(rng, n):
    return rng.integers(I64_MIN, I64_MAX, n, dtype=np.int64, endpoint=True)


@pytest.mark.parametrize("n", [1 << 18, (1 << 18) + 12345, 1_000_003, 4_000_000])
def test_uniform_full_range(n):
    rng = np.random.default_rng(n)
    keys = full_range(rng, n)
    for desc in (False, True):
        check_sort(keys, desc)


def test_cfg2_shape_duplicates():
    """cfg2's generator (~1% duplicates copied from earlier rows) at 2M rows."""
    rng = np.random.default_rng(0)
    n = 2_000_000
    keys = full_range(rng, n)
    dst = rng.choice(np.arange(1, n), n // 100, replace=False)
    src = (rng.random(n // 100) * dst).astype(np.int64)
    keys[dst] = keys[src]
    check_sort(keys)
    check_sort(keys, True)


def test_heavy_duplicates_equal_subbuckets():
    """Few distinct wide values: sub-buckets of equal keys (copy branch)."""
    rng = np.random.default_rng(5)
    vals = full_range(rng, 3000)
    keys = vals[rng.integers(0, 3000, 1_000_000)]
    check_sort(keys)
    check_sort(keys, True)


def test_large_bins_bitonic_branch():
    """Sub-buckets whose top varying byte leaves > 16 rows per digit with
    distinct low bits (warp bitonic by (key, row id)), with repeats."""
    rng = np.random.default_rng(6)
    n_groups, per = 2000, 300
    tops = full_range(rng, n_groups) & ~np.int64((1 << 48) - 1)
    parts = []
    for g in range(n_groups):
        low = rng.integers(0, 1 << 40, per, dtype=np.int64)
        low[:5] |= np.int64(1) << 47  # top varying bit 47 -> digit bits 40..47; the rest share digit 0
        low[per // 2:per // 2 + 40] = low[per // 2]  # equal keys inside the big bin
        parts.append(tops[g] | low)
    keys = np.concatenate(parts)
    keys = keys[rng.permutation(len(keys))]
    # plus uniform background so the top digits pass the spread pre-check
    keys = np.concatenate([keys, full_range(rng, 1_000_000)])
    check_sort(keys)
    check_sort(keys, True)


def test_small_bins_insertion_branch():
    """Rows differing only below the top varying byte, a few per digit."""
    rng = np.random.default_rng(7)
    base = full_range(rng, 400_000)
    extra = base[rng.integers(0, len(base), 200_000)] ^ rng.integers(0, 1 << 12, 200_000, dtype=np.int64)
    check_sort(np.concatenate([base, extra]))


def test_precheck_fallback_narrow_keys():
    """Top 16 bits constant (keys in [0, 2^40)): the pre-check hands over to LSD."""
    rng = np.random.default_rng(8)
    keys = rng.integers(0, 1 << 40, 1_500_000, dtype=np.int64)
    check_sort(keys)
    check_sort(keys, True)


def test_overflow_fallback_after_passes():
    """Spread top digits but one sub-bucket above the on-chip cap: detected
    after the two passes, the LSD kernel behind it produces the result."""
    rng = np.random.default_rng(9)
    n = 1_000_000
    keys = full_range(rng, n)
    hot = np.int64(0x1234) << 48
    keys[rng.choice(n, LOCAL_CAP + 1200, replace=False)] = hot | rng.integers(0, 1 << 48, LOCAL_CAP + 1200,
                                                                           dtype=np.int64)
    check_sort(keys)
    check_sort(keys, True)


def test_extremes_and_sign_boundary():
    rng = np.random.default_rng(10)
    keys = full_range(rng, 600_000)
    keys[::97] = I64_MIN
    keys[::89] = I64_MAX
    keys[::83] = -1
    keys[::79] = 0
    check_sort(keys)
    check_sort(keys, True)


def test_hybrid_matches_forced_lsd(monkeypatch):
    """Same permutation from the hybrid and the LSD path (RL_NO_HYBRID)."""
    rng = np.random.default_rng(11)
    keys = full_range(rng, 3_000_000)
    kd = torch.from_numpy(keys).cuda()
    a = engine.sort_permutation([engine.SortAxis(kd, False)], len(keys), kd.device)
    monkeypatch.setenv("RL_NO_HYBRID", "1")
    b = engine.sort_permutation([engine.SortAxis(kd, False)], len(keys), kd.device)
    assert torch.equal(a, b)


@pytest.mark.parametrize("width", [4, 8, 5])
@pytest.mark.parametrize("shape", ["uniform", "bitonic_bins"])
def test_fused_gather_in_local_phase(width, shape):
    """Relation.take fused into the hybrid's local phase: one 4- or 8-byte
    column takes the prefetch-and-park path, other widths the direct loads;
    bins sorted by the bitonic network reload their moved rows."""
    rng = np.random.default_rng(12 + width)
    if shape == "uniform":
        keys = full_range(rng, 1_500_000)
    else:
        tops = full_range(rng, 500) & ~np.int64((1 << 48) - 1)
        low = rng.integers(0, 1 << 40, (500, 200), dtype=np.int64)
        low[:, :3] |= np.int64(1) << 47
        keys = np.concatenate([(tops[:, None] | low).ravel(), full_range(rng, 800_000)])
        keys = keys[rng.permutation(len(keys))]
    n = len(keys)
    col = rng.integers(0, 256, (n, width), dtype=np.uint8)
    kd = torch.from_numpy(keys).cuda()
    cd = torch.from_numpy(col).cuda()
    out = torch.empty_like(cd)
    perm = engine.sort_permutation([engine.SortAxis(kd, False)], n, kd.device,
                                   gather=[engine.OutColumn(cd, out, width, 0)], fuse_gather=True)
    want = O.stable_axis_order(keys, False)
    assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == want).all()
    assert (out.cpu().numpy() == col[want]).all()


def test_chunk_counter_wrap_fallback():
    """> 65535 rows of one sub-bucket inside one scatter chunk (10M rows, the
    first 1M in sub-bucket 0x8123): the chunk's 16-bit counter wraps, the LSD
    fallback recounts digits 6 and 7 itself."""
    rng = np.random.default_rng(13)
    n = 10_000_000
    keys = full_range(rng, n)
    keys[:1_000_000] = (np.int64(0x0123) << 48) | rng.integers(0, 1 << 48, 1_000_000, dtype=np.int64)
    check_sort(keys)


def test_scatter_cfg2_size_with_ties():
    """cfg2's size (10M) with cfg2's duplicate pattern, both directions."""
    rng = np.random.default_rng(14)
    n = 10_000_000
    keys = full_range(rng, n)
    dst = rng.choice(np.arange(1, n), n // 100, replace=False)
    src = (rng.random(n // 100) * dst).astype(np.int64)
    keys[dst] = keys[src]
    check_sort(keys)
    check_sort(keys, True)


@pytest.mark.parametrize("tops", [(0x10, 0x90), (0x7F,)])
def test_split_digit7_buckets(tops):
    """Digit 7 takes one or two values, digit 6 spreads: every digit-7 bucket
    holds far more than one pass-B work item, so it is cut at chunk
    boundaries and later slices start from the earlier chunks' counts."""
    rng = np.random.default_rng(15 + len(tops))
    n = 500_000 * len(tops)
    hi = np.array(tops, dtype=np.int64)[rng.integers(0, len(tops), n)]
    keys = (hi << np.int64(56)) | rng.integers(0, 1 << 56, n, dtype=np.int64)
    check_sort(keys)
    check_sort(keys, True)


@pytest.mark.parametrize("bits,n", [(27, 5_000_000), (33, 4_500_000), (40, 6_000_000)])
def test_scatter_narrow_keys_shifted(bits, n):
    """Keys with constant leading bits (row-id-like, in [0, 2^bits) plus an
    offset and negatives): the scatter path shifts the constant prefix out
    (top 16 VARYING bits as sub-buckets) and restores it on output."""
    rng = np.random.default_rng(40 + bits)
    keys = rng.integers(0, 1 << bits, n, dtype=np.int64) - (1 << (bits - 1)) + 123_456_789
    keys[rng.choice(n, n // 50, replace=False)] = keys[rng.integers(0, n, n // 50)]  # duplicates
    check_sort(keys)
    check_sort(keys, True)


def test_scatter_shift_missed_by_sample():
    """A single key varying in a high bit the sample does not see: the chunk
    counts catch it and the LSD passes produce the (identical) result."""
    rng = np.random.default_rng(44)
    n = 6_000_001
    keys = rng.integers(0, 1 << 30, n, dtype=np.int64)
    keys[3] = np.int64(1) << 50  # not at a sampled position
    check_sort(keys)


@pytest.mark.parametrize("shape", ["composite", "low_zero_bits", "three_runs"])
def test_scatter_packed_keys(shape):
    """Varying bits in two runs (cfg4's (a << 32) | b with 16-bit parts), keys
    with constant low bits (multiples of 64), and three runs (not packed:
    the keys are used as they are) — all equal to the stable argsort."""
    rng = np.random.default_rng(50 + len(shape))
    n = 4_500_000
    if shape == "composite":
        a = rng.integers(0, 2**16, n).astype(np.int64)
        b = rng.integers(0, 2**16, n).astype(np.int64)
        keys = (a << np.int64(32)) | b
    elif shape == "low_zero_bits":
        keys = rng.integers(-(1 << 33), 1 << 33, n, dtype=np.int64) * 64
    else:
        keys = ((rng.integers(0, 2**12, n).astype(np.int64) << np.int64(50))
                | (rng.integers(0, 2**12, n).astype(np.int64) << np.int64(30))
                | rng.integers(0, 2**12, n).astype(np.int64))
    check_sort(keys)
    check_sort(keys, True)


@pytest.mark.parametrize("n", [1 << 18, 1_500_000])
def test_hybrid_then_lsd_same_size(n):
    """A wide-key sort (hybrid) then sorts the cooperative kernel must take LSD
    (narrow keys: too few varying digits; one huge sub-bucket) on the same
    workspace. The sub-bucket table is stale from the first sort, so the local
    phase must see the LSD sort's "no local phase" signal and not run."""
    rng = np.random.default_rng(n + 7)
    check_sort(full_range(rng, n))
    check_sort(rng.integers(0, 1 << 20, n, dtype=np.int64))  # three varying digits: LSD
    check_sort(np.where(rng.random(n) < 0.5, 5, full_range(rng, n)).astype(np.int64))  # skew: fallback
    check_sort(full_range(rng, n))


@pytest.mark.parametrize("packed", ["on", "off"])
@pytest.mark.parametrize("bits", [20, 30, 32])
def test_scatter_packed_rows(packed, bits, monkeypatch, into_subbuckets):
    """Keys with <= 32 varying bits travel with their row id in ONE u64 word
    (packed rows: no row-id stream in the counting passes and the local phase).
    The result equals the stable argsort with the mode on and forced off
    (RL_NO_PACKED_ROWS=1), ties (duplicates) included, both directions, with a
    fused gather riding on the packed row ids."""
    if packed == "off":
        monkeypatch.setenv("RL_NO_PACKED_ROWS", "1")
    rng = np.random.default_rng(60 + bits)
    n = 5_000_000 if into_subbuckets == "scatter" else 1_500_000
    keys = rng.integers(0, 1 << bits, n, dtype=np.int64) - (1 << (bits - 1)) + 987_654_321
    keys[rng.choice(n, n // 20, replace=False)] = keys[rng.integers(0, n, n // 20)]
    check_sort(keys)
    check_sort(keys, True)
    col = rng.integers(0, 256, (n, 8), dtype=np.uint8)
    kd, cd = torch.from_numpy(keys).cuda(), torch.from_numpy(col).cuda()
    out = torch.empty_like(cd)
    perm = engine.sort_permutation([engine.SortAxis(kd, False)], n, kd.device,
                                   gather=[engine.OutColumn(cd, out, 8, 0)], fuse_gather=True)
    want = O.stable_axis_order(keys, False)
    assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == want).all()
    assert (out.cpu().numpy() == col[want]).all()


@pytest.mark.parametrize("bits", [30, 64])
def test_three_level_scatter(bits, monkeypatch, into_subbuckets):
    """The third level (digit 5 inside every (d7, d6) sub-bucket, the local
    phase over 2^24 sub-sub-buckets) forced at a small size with
    RL_LEVEL3_MIN_ROWS: narrow (packed-row) and full-range keys, duplicates,
    both directions, a fused gather — equal to the stable argsort."""
    if into_subbuckets != "scatter":
        pytest.skip("the third level belongs to the scatter path")
    monkeypatch.setenv("RL_LEVEL3_MIN_ROWS", "1")
    rng = np.random.default_rng(70 + bits)
    n = 3_000_000
    keys = full_range(rng, n) if bits == 64 else rng.integers(0, 1 << bits, n, dtype=np.int64)
    keys[rng.choice(n, n // 30, replace=False)] = keys[rng.integers(0, n, n // 30)]
    check_sort(keys)
    check_sort(keys, True)
    col = rng.integers(0, 256, (n, 4), dtype=np.uint8)
    kd, cd = torch.from_numpy(keys).cuda(), torch.from_numpy(col).cuda()
    out = torch.empty_like(cd)
    perm = engine.sort_permutation([engine.SortAxis(kd, False)], n, kd.device,
                                   gather=[engine.OutColumn(cd, out, 4, 0)], fuse_gather=True)
    want = O.stable_axis_order(keys, False)
    assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == want).all()
    assert (out.cpu().numpy() == col[want]).all()


def test_three_level_skewed_sub_sub_bucket_falls_back(monkeypatch, into_subbuckets):
    """A sub-sub-bucket above the on-chip cap: the LSD fallback, same result."""
    if into_subbuckets != "scatter":
        pytest.skip("the third level belongs to the scatter path")
    monkeypatch.setenv("RL_LEVEL3_MIN_ROWS", "1")
    rng = np.random.default_rng(77)
    n = 2_000_000
    keys = full_range(rng, n)
    keys[:5000] = (keys[:5000] & ~np.int64((1 << 40) - 1)) | rng.integers(0, 1 << 40, 5000)  # one 24-bit prefix
    keys[:5000] = (np.int64(0x123456) << np.int64(40)) | rng.integers(0, 1 << 40, 5000)
    check_sort(keys)


@pytest.mark.parametrize("shape", ["narrow_2cols", "narrow_mixed", "wide_keys_fallback", "three_level", "idw_4b",
                                   "idw_2x2b_dups", "idw_3b_three_level", "idw_heavy_bins"])
def test_sort_with_carried_columns(shape, monkeypatch, into_subbuckets):
    """rl_sort_axis_carry: the other columns ride with the packed rows through
    the counting passes and leave from each run's payload window — equal to
    the stable argsort + take; wide keys take the LSD fallback with the
    gathers fused; the third level forced at a small size. idw: keys that do
    not pack with <= 4 carried bytes share one word with the row id (cfg2's
    shape: full-range keys + a 4-byte payload), incl. duplicate-heavy bins
    (equal keys ranked by the ids behind the load indexes, bitonic bins)."""
    if into_subbuckets != "scatter":
        pytest.skip("carried columns belong to the scatter path")
    if "three_level" in shape:
        monkeypatch.setenv("RL_LEVEL3_MIN_ROWS", "1")
    rng = np.random.default_rng(90 + len(shape))
    n = 4_500_000
    if shape == "wide_keys_fallback" or shape.startswith("idw"):
        keys = full_range(rng, n)
        if shape == "idw_2x2b_dups":
            keys[rng.choice(n, n // 10, replace=False)] = keys[rng.integers(0, n, n // 10)]
        if shape == "idw_heavy_bins":  # bins of ~40 equal keys (the warp bitonic) and of 2-32 (the rank loop)
            keys[: n // 2] = keys[rng.integers(0, n // 80, n // 2)]
            rng.shuffle(keys)
    else:
        keys = rng.integers(0, 1 << 27, n, dtype=np.int64) - 5_000_000
        keys[rng.choice(n, n // 25, replace=False)] = keys[rng.integers(0, n, n // 25)]
    if shape == "narrow_mixed":
        cols = [rng.integers(0, 256, (n, 5), dtype=np.uint8), rng.integers(-(2**31), 2**31, n).astype(np.int32),
                rng.integers(0, 256, (n, 3), dtype=np.uint8)]
    elif shape in ("idw_4b", "idw_heavy_bins"):
        cols = [rng.integers(-(2**31), 2**31, n).astype(np.int32)]
    elif shape == "idw_2x2b_dups":
        cols = [rng.integers(0, 256, (n, 2), dtype=np.uint8), rng.integers(0, 256, (n, 2), dtype=np.uint8)]
    elif shape == "idw_3b_three_level":
        cols = [rng.integers(0, 256, (n, 3), dtype=np.uint8)]
    else:
        cols = [rng.integers(-(2**62), 2**62, n), rng.integers(-(2**62), 2**62, n)]
    for desc in (False, True):
        kd = torch.from_numpy(keys).cuda()
        srcs = [torch.from_numpy(c).cuda() for c in cols]
        w = lambda c: c.element_size() * (c.shape[1] if c.dim() > 1 else 1)  # noqa: E731
        outs = [engine.OutColumn(c, torch.empty_like(c), w(c), 0) for c in srcs]
        sk = torch.empty_like(kd)
        perm = engine.sort_carry(kd, desc, sk, outs)
        want = O.stable_axis_order(keys, desc)
        assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == want).all()
        assert (sk.cpu().numpy() == keys[want]).all()
        for o, c in zip(outs, cols):
            assert (o.dst.cpu().numpy() == c[want]).all()


def test_sort_graph_carried_payload_equals_gather(into_subbuckets):
    """engine.SortGraph with the 4-byte payload carried through the passes
    (idw) replays to the same sorted keys, permutation and payload as the
    sort + gather graph (cfg2's shape at 5M rows, ~1% duplicates)."""
    if into_subbuckets != "scatter":
        pytest.skip("carried columns belong to the scatter path")
    from paper_2602_21237_b200 import synth

    rel = synth.cfg2_relation(5_000_000)
    keys = torch.from_numpy(rel.column("key").copy()).cuda()
    pay = torch.from_numpy(np.ascontiguousarray(rel.column("payload")).view(np.int32).reshape(-1).copy()).cuda()
    got = []
    for carry in (False, True):
        dst = torch.empty_like(pay)
        g = engine.SortGraph(keys, gather=[engine.OutColumn(pay, dst, 4, 0)], carry=carry)
        assert g.carry == carry
        for _ in range(2):
            dst.zero_()
            g.replay()
        torch.cuda.synchronize()
        got.append((g.sorted_keys.cpu(), g.perm.cpu(), dst.cpu()))
    want = O.stable_axis_order(rel.column("key"), False)
    assert (got[1][1].numpy().view(np.uint32).astype(np.int64) == want).all()
    for a, b in zip(*got):
        assert torch.equal(a, b)
