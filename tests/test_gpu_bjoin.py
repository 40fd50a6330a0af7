"""The bucket join (csrc/bucket_join.cu) against the oracle and the sort-based
plan: the same pair count, the same output rows in the same (key, left row,
right row) order (tensorpath.py:149-185), chunked slices, the pair checksum,
and the cases where it must decline (keys needing more than 32 bits, skewed
sub-buckets) and leave the join to the sort-based plan."""

import numpy as np
import pytest
import torch

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import _capi as C
from paper_2602_21237_b200 import engine, pipeline

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["listed", "sorted"])
def emit_path(request, monkeypatch):
    """Every test twice: runs with few pairs listing their matches (the
    default for <= 512 pairs a run) and every run sorting both sides
    (RL_BJ_NO_SEL=1)."""
    if request.param == "sorted":
        monkeypatch.setenv("RL_BJ_NO_SEL", "1")
    else:
        monkeypatch.delenv("RL_BJ_NO_SEL", raising=False)
    return request.param


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _pairs(plan, a=0, b=None):
    b = plan.total if b is None else b
    lr = torch.empty(max(b - a, 1), dtype=torch.int32, device="cuda")
    rr = torch.empty(max(b - a, 1), dtype=torch.int32, device="cuda")
    if b > a:
        plan.expand(a, b, (), lr[: b - a], rr[: b - a])
    u = lambda t: t[: b - a].cpu().numpy().view(np.uint32).astype(np.int64)  # noqa: E731
    return u(lr), u(rr)


def _check(lk, rk, expect_bucket=True):
    bp = engine.BucketJoinPlan(_dev(lk), _dev(rk))
    assert bp.applies == expect_bucket
    if not expect_bucket:
        return bp
    wl, wr = O.join_pairs(lk, rk)
    assert bp.total == len(wl)
    gl, gr = _pairs(bp)
    assert (gl == wl).all() and (gr == wr).all()
    acc = torch.zeros(1, dtype=torch.int64, device="cuda")
    bp.pair_checksum(0, bp.total, acc)
    assert int(acc.item()) & (2**64 - 1) == O.pair_checksum(wl, wr)
    return bp


@pytest.mark.parametrize("n,dom", [(1_000_000, 1_000_000), (300_000, 50_000), (200_000, 3_000), (1 << 16, 1 << 30)])
def test_uniform_joins_match_the_oracle(n, dom):
    rng = np.random.default_rng(n + dom)
    _check(rng.integers(0, dom, n), rng.integers(0, dom, n + 12345))


def test_negative_keys_and_unequal_sides():
    rng = np.random.default_rng(3)
    lk = rng.integers(-80_000, -1, 400_000)  # all negative: high bits constant (two's complement)
    rk = rng.integers(-90_000, -10_000, 90_000)
    _check(lk, rk)
    _check(rk, lk)
    # keys crossing zero vary in every bit (bit masks cannot pack them): the plan declines
    _check(rng.integers(-40_000, 40_000, 400_000), rng.integers(-10_000, 70_000, 90_000), expect_bucket=False)


def test_composite_two_runs_cfg4_shape():
    rng = np.random.default_rng(4)
    n = 500_000
    mk = lambda: (rng.integers(0, 2**8, n).astype(np.int64) << np.int64(32)) | rng.integers(0, 2**8, n)  # noqa: E731
    _check(mk(), mk())


def test_no_matches_and_single_key_groups():
    rng = np.random.default_rng(5)
    lk = rng.integers(0, 1 << 20, 200_000) * 2
    _check(lk, lk + 1)  # disjoint: total 0


def test_heavy_duplicates_fit_then_fall_back():
    rng = np.random.default_rng(6)
    # ~40 rows per key on each side: big pair counts per run, still within the sub-bucket cap
    keys = rng.integers(0, 20_000, 800_000)
    bp = _check(keys, rng.integers(0, 20_000, 600_000))
    assert bp.total > 10**7
    # one key holding 10% of the rows: its sub-bucket exceeds the cap -> decline
    skew = rng.integers(0, 1_000_000, 500_000)
    skew[::10] = 77
    _check(skew, rng.integers(0, 1_000_000, 500_000), expect_bucket=False)


def test_wide_keys_decline():
    rng = np.random.default_rng(7)
    lk = rng.integers(-(2**62), 2**62, 300_000)
    _check(lk, lk[::3].copy(), expect_bucket=False)


def test_varying_bit_missed_by_the_joint_sample():
    rng = np.random.default_rng(8)
    lk = rng.integers(0, 1 << 20, 300_001)
    rk = rng.integers(0, 1 << 20, 300_001)
    rk[5] = 1 << 40  # a bit the sample misses: the chunk counts catch it
    _check(lk, rk, expect_bucket=False)


def test_chunked_slices_and_columns():
    rng = np.random.default_rng(9)
    n = 400_000
    lk, rk = rng.integers(0, 100_000, n), rng.integers(0, 100_000, n)
    lp = rng.integers(0, 256, (n, 5), dtype=np.uint8)
    rp = rng.integers(-(2**40), 2**40, n)
    bp = engine.BucketJoinPlan(_dev(lk), _dev(rk))
    assert bp.applies
    wl, wr = O.join_pairs(lk, rk)
    for a, b in [(0, 1), (17, 100_003), (bp.total // 2, bp.total), (bp.total - 5, bp.total)]:
        gl, gr = _pairs(bp, a, b)
        assert (gl == wl[a:b]).all() and (gr == wr[a:b]).all()
    total = bp.total
    cols = [engine.OutColumn(None, torch.empty(total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_KEY),
            engine.OutColumn(_dev(lp), torch.empty((total, 5), dtype=torch.uint8, device="cuda"), 5, C.RL_SIDE_LEFT),
            engine.OutColumn(_dev(rp), torch.empty(total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_RIGHT)]
    bp.expand(0, total, cols)
    assert (cols[0].dst.cpu().numpy() == lk[wl]).all()
    assert (cols[1].dst.cpu().numpy() == lp[wl]).all()
    assert (cols[2].dst.cpu().numpy() == rp[wr]).all()


def test_pipeline_join_uses_the_bucket_plan_and_equals_the_sort_plan(monkeypatch):
    rng = np.random.default_rng(10)
    n = 5_000_000  # above the bucket join's 4M-row threshold
    lk, rk = rng.integers(0, n, n), rng.integers(0, n, n)
    plan = pipeline.plan_join(_dev(lk), _dev(rk))
    assert plan.kind == "bucket"
    monkeypatch.setenv("RL_NO_BJOIN", "1")
    plan2 = pipeline.plan_join(_dev(lk), _dev(rk))
    assert plan2.kind == "sort" and plan2.total == plan.total
    a, b = _pairs(plan)
    c, d = _pairs(plan2)
    assert (a == c).all() and (b == d).all()


def test_small_inputs_forced(monkeypatch):
    monkeypatch.setenv("RL_FORCE_BJOIN", "1")
    rng = np.random.default_rng(11)
    for nl, nr, dom in [(1, 1, 1), (1, 50, 3), (7, 3, 2), (1000, 800, 100), (5000, 1, 10)]:
        _check(rng.integers(0, dom, nl), rng.integers(0, dom, nr))


@pytest.mark.parametrize("shape", ["int64", "bytes16", "mixed3", "too_wide"])
def test_carried_payload_columns(shape):
    """Payload columns carried with the rows through the partition passes
    (<= 16 bytes a side, natural alignment) come out exactly as the gathered
    ones; wider payloads fall back to gathering by row id."""
    rng = np.random.default_rng(20 + len(shape))
    n = 600_000
    lk, rk = rng.integers(0, 300_000, n), rng.integers(0, 300_000, n - 999)
    if shape == "int64":
        lc = [rng.integers(-(2**62), 2**62, n)]
        rc = [rng.integers(-(2**62), 2**62, n - 999)]
    elif shape == "bytes16":
        lc = [rng.integers(0, 256, (n, 16), dtype=np.uint8)]
        rc = [rng.integers(0, 256, (n - 999, 16), dtype=np.uint8)]
    elif shape == "mixed3":
        lc = [rng.integers(0, 256, (n, 3), dtype=np.uint8), rng.integers(-5, 5, n),
              rng.integers(0, 256, (n, 4), dtype=np.uint8)]
        rc = [rng.integers(0, 256, (n - 999, 1), dtype=np.uint8)]
    else:
        lc = [rng.integers(0, 256, (n, 24), dtype=np.uint8)]
        rc = [rng.integers(0, 256, (n - 999, 12), dtype=np.uint8), rng.integers(0, 9, n - 999)]
    ldev, rdev = [_dev(c) for c in lc], [_dev(c) for c in rc]
    bp = engine.BucketJoinPlan(_dev(lk), _dev(rk), ldev, rdev)
    assert bp.applies
    wl, wr = O.join_pairs(lk, rk)
    assert bp.total == len(wl)
    w = lambda c: c.element_size() * (c.shape[1] if c.dim() > 1 else 1)  # noqa: E731
    cols = [engine.OutColumn(None, torch.empty(bp.total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_KEY)]
    cols += [engine.OutColumn(c, torch.empty((bp.total,) + tuple(c.shape[1:]), dtype=c.dtype, device="cuda"), w(c),
                              C.RL_SIDE_LEFT) for c in ldev]
    cols += [engine.OutColumn(c, torch.empty((bp.total,) + tuple(c.shape[1:]), dtype=c.dtype, device="cuda"), w(c),
                              C.RL_SIDE_RIGHT) for c in rdev]
    half = bp.total // 3
    bp.expand(0, half, [engine.OutColumn(c.src, c.dst[:half], c.width, c.side) for c in cols])
    bp.expand(half, bp.total, [engine.OutColumn(c.src, c.dst[half:], c.width, c.side) for c in cols])
    assert (cols[0].dst.cpu().numpy() == lk[wl]).all()
    for c, h in zip(cols[1:1 + len(lc)], lc):
        assert (c.dst.cpu().numpy() == h[wl]).all()
    for c, h in zip(cols[1 + len(lc):], rc):
        assert (c.dst.cpu().numpy() == h[wr]).all()
    expect_words = {"int64": 1, "bytes16": 2, "mixed3": 2, "too_wide": 0}[shape]
    assert bp.plan.words_left == expect_words


@pytest.mark.parametrize("carry", [False, True])
def test_three_level_partition(carry, monkeypatch):
    """The bucket join over 2^24 sub-sub-buckets (the partition's third level,
    forced at this size with RL_BJ_LEVELS=3): same pairs, order, columns and
    checksum as the oracle, payload carried through the digit-5 pass too."""
    monkeypatch.setenv("RL_BJ_LEVELS", "3")
    rng = np.random.default_rng(31)
    n = 3_000_000
    lk, rk = rng.integers(0, 2_000_000, n), rng.integers(0, 2_000_000, n + 7)
    bp = _check(lk, rk)
    assert bp.plan.levels == 3
    lp = rng.integers(-(2**60), 2**60, n)
    rp = rng.integers(0, 256, (n + 7, 12), dtype=np.uint8)
    ld, rd = _dev(lp), _dev(rp)
    bp = engine.BucketJoinPlan(_dev(lk), _dev(rk), [ld] if carry else [], [rd] if carry else [])
    wl, wr = O.join_pairs(lk, rk)
    cols = [engine.OutColumn(None, torch.empty(bp.total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_KEY),
            engine.OutColumn(ld, torch.empty(bp.total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_LEFT),
            engine.OutColumn(rd, torch.empty((bp.total, 12), dtype=torch.uint8, device="cuda"), 12, C.RL_SIDE_RIGHT)]
    bp.expand(0, bp.total, cols)
    assert bp.plan.words_left == (1 if carry else 0) and bp.plan.words_right == (2 if carry else 0)
    assert (cols[0].dst.cpu().numpy() == lk[wl]).all()
    assert (cols[1].dst.cpu().numpy() == lp[wl]).all()
    assert (cols[2].dst.cpu().numpy() == rp[wr]).all()


def test_strided_outputs_and_split_gather():
    """rl_bjoin_expand_strided writes 8-byte columns row-interleaved exactly as
    the plain expand writes them apart; bad strides / alignment are refused;
    rl_gather_rows_split16 takes interleaved rows into two columns."""
    rng = np.random.default_rng(41)
    n = 300_000
    lk, rk = rng.integers(0, 150_000, n), rng.integers(0, 150_000, n)
    lp, rp = rng.integers(-(2**50), 2**50, n), rng.integers(-(2**50), 2**50, n)
    bp = engine.BucketJoinPlan(_dev(lk), _dev(rk), [_dev(lp)], [_dev(rp)])
    assert bp.applies
    t = bp.total
    wl, wr = O.join_pairs(lk, rk)
    key = torch.empty(t, dtype=torch.int64, device="cuda")
    inter = torch.empty((t, 16), dtype=torch.uint8, device="cuda")
    cols = [engine.OutColumn(None, key, 8, C.RL_SIDE_KEY),
            engine.OutColumn(_dev(lp), inter[:, :8], 8, C.RL_SIDE_LEFT),
            engine.OutColumn(_dev(rp), inter[:, 8:], 8, C.RL_SIDE_RIGHT)]
    bp.expand(0, t, cols, dst_strides=[0, 16, 16])
    both = inter.cpu().numpy().view(np.int64).reshape(t, 2)
    assert (key.cpu().numpy() == lk[wl]).all()
    assert (both[:, 0] == lp[wl]).all() and (both[:, 1] == rp[wr]).all()
    with pytest.raises(ValueError):  # stride below the width
        bp.expand(0, t, cols, dst_strides=[0, 4, 16])
    with pytest.raises(ValueError):  # a 5-byte column cannot be interleaved
        odd = torch.empty((t, 16), dtype=torch.uint8, device="cuda")
        bp.expand(0, t, [engine.OutColumn(_dev(rng.integers(0, 256, (n, 5), dtype=np.uint8)), odd, 5,
                                          C.RL_SIDE_LEFT)], dst_strides=[16])
    perm = torch.from_numpy(rng.permutation(t).astype(np.int32)).cuda()
    lo = torch.empty(t, dtype=torch.int64, device="cuda")
    hi = torch.empty(t, dtype=torch.int64, device="cuda")
    engine.gather_split16(perm, inter, lo, hi)
    p = perm.cpu().numpy().astype(np.int64)
    assert (lo.cpu().numpy() == both[p, 0]).all() and (hi.cpu().numpy() == both[p, 1]).all()
    with pytest.raises(ValueError):  # source rows must be 16-byte aligned
        engine.gather_split16(perm, inter.view(-1)[8:8 + 16 * (t - 1)].view(t - 1, 16), lo, hi)
    engine.gather_split16(perm[:0], inter, lo, hi)  # m = 0: nothing to do


def test_selective_join_listed_runs(emit_path):
    """A selective join (~0.05 pairs a row: every run lists its few matches
    unless RL_BJ_NO_SEL=1): pairs, order, slices, checksum and carried /
    gathered columns equal the oracle."""
    rng = np.random.default_rng(43)
    n = 1_000_000
    lk, rk = rng.integers(0, 20_000_000, n), rng.integers(0, 20_000_000, n + 333)
    bp = _check(lk, rk)
    wl, wr = O.join_pairs(lk, rk)
    for a, b in [(0, 7), (1000, bp.total - 1000)]:
        gl, gr = _pairs(bp, a, b)
        assert (gl == wl[a:b]).all() and (gr == wr[a:b]).all()
    lp = rng.integers(-(2**62), 2**62, n)
    rp = rng.integers(0, 256, (n + 333, 16), dtype=np.uint8)
    bc = engine.BucketJoinPlan(_dev(lk), _dev(rk), [_dev(lp)], [])
    cols = [engine.OutColumn(None, torch.empty(bc.total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_KEY),
            engine.OutColumn(_dev(lp), torch.empty(bc.total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_LEFT),
            engine.OutColumn(_dev(rp), torch.empty((bc.total, 16), dtype=torch.uint8, device="cuda"), 16,
                             C.RL_SIDE_RIGHT)]
    bc.expand(0, bc.total, cols)
    assert (cols[0].dst.cpu().numpy() == lk[wl]).all()
    assert (cols[1].dst.cpu().numpy() == lp[wl]).all()
    assert (cols[2].dst.cpu().numpy() == rp[wr]).all()


@pytest.mark.parametrize("levels", [2, 3])
def test_mixed_dense_and_selective_runs(levels, emit_path, monkeypatch):
    """One plan holding both kinds of run: the lower half of the key range is
    ~24 rows a key on each side (dense runs: rows binned and ranked), the
    upper half ~0.1 matches a row (selective runs: matches listed by the
    count kernel, the 1/8 rule per run). Pairs, order, slices that start and
    end inside either kind, checksum and gathered columns equal the oracle,
    over the two- and the three-level partition."""
    if levels == 3:
        monkeypatch.setenv("RL_BJ_LEVELS", "3")
    rng = np.random.default_rng(47 + levels)
    half = 200_000

    def side(m):
        dense = rng.integers(0, 1 << 13, m) * 256  # 8192 keys below 2^21
        sparse = rng.integers(1 << 21, 1 << 22, m + 17)  # 2M keys above it
        k = np.concatenate([dense, sparse])
        return k[rng.permutation(len(k))]

    lk, rk = side(half), side(half + 101)
    bp = _check(lk, rk)
    if levels == 3:
        assert bp.plan.levels == 3
    wl, wr = O.join_pairs(lk, rk)
    dense_pairs = int((lk[wl] < (1 << 21)).sum())
    assert 0 < dense_pairs < bp.total  # both kinds of run produced pairs
    first_sparse = int(np.argmax(lk[wl] >= (1 << 21)))
    for a, b in [(first_sparse - 5, first_sparse + 9), (3, bp.total - 3), (bp.total - 1, bp.total)]:
        gl, gr = _pairs(bp, a, b)
        assert (gl == wl[a:b]).all() and (gr == wr[a:b]).all()
    rp = rng.integers(0, 256, (len(rk), 8), dtype=np.uint8)
    cols = [engine.OutColumn(None, torch.empty(bp.total, dtype=torch.int64, device="cuda"), 8, C.RL_SIDE_KEY),
            engine.OutColumn(_dev(rp), torch.empty((bp.total, 8), dtype=torch.uint8, device="cuda"), 8,
                             C.RL_SIDE_RIGHT)]
    bp.expand(0, bp.total, cols)
    assert (cols[0].dst.cpu().numpy() == lk[wl]).all()
    assert (cols[1].dst.cpu().numpy() == rp[wr]).all()
