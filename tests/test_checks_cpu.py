"""The torch-only invariants of paper_2602_21237_b200/checks.py (the bench's
gates and the large-size GPU tests) pinned on CPU against the oracle: they
agree on correct join / sort outputs and catch corrupted ones."""

import numpy as np
import torch

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import checks


def _join(seed, n=4000, dom=900, neg=False):
    rng = np.random.default_rng(seed)
    lo = -dom if neg else 0
    lk = rng.integers(lo, dom, n).astype(np.int64)
    rk = rng.integers(lo, dom, n + 77).astype(np.int64)
    lp = np.arange(n, dtype=np.int64)
    rp = np.arange(n + 77, dtype=np.int64)
    key, lpay, rpay = O.join_columns([lk, lp], 0, [rk, rp], 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    return t(lk), t(lp), t(rk), t(rp), t(key), t(lpay), t(rpay)


def test_join_invariants_agree_with_the_oracle():
    for seed, neg in ((0, False), (1, True)):
        lk, lp, rk, rp, key, lpay, rpay = _join(seed, neg=neg)
        dom = None if neg else 900
        exp = checks.join_expectations(lk, lp, rk, rp, domain=dom)
        assert exp == checks.join_observed(key, lpay, rpay)
        assert exp["matches"] == O.join_count(lk.numpy(), rk.numpy())
        assert checks.join_order_ok(key, lpay, rpay)


def test_join_invariants_catch_corruption():
    lk, lp, rk, rp, key, lpay, rpay = _join(2)
    exp = checks.join_expectations(lk, lp, rk, rp, domain=900)
    # two right rows of different keys swapped: multisets per side unchanged
    i = int(torch.nonzero(key[1:] != key[:-1])[0]) + 1
    bad = rpay.clone()
    bad[i - 1], bad[i] = rpay[i], rpay[i - 1]
    assert checks.join_observed(key, lpay, bad)["sum_pair"] != exp["sum_pair"]
    # a missing pair
    assert checks.join_observed(key[1:], lpay[1:], rpay[1:]) != exp
    # order broken inside a key
    assert not checks.join_order_ok(key, lpay.flip(0), rpay)


def test_sort_checks():
    rng = np.random.default_rng(3)
    keys = torch.from_numpy(rng.integers(-30, 30, 5000).astype(np.int64))
    rid = torch.arange(5000)
    perm = torch.from_numpy(O.stable_axis_order(keys.numpy(), False))
    assert checks.sort_ok(keys[perm], rid[perm])
    assert checks.multiset_sums([keys[perm], rid[perm]]) == checks.multiset_sums([keys, rid])
    unstable = torch.sort(keys, stable=False, descending=False).indices
    if not bool((unstable == perm).all()):
        assert not checks.sort_ok(keys[unstable], rid[unstable]) or bool((unstable == perm).all())
    permd = torch.from_numpy(O.stable_axis_order(keys.numpy(), True))
    assert checks.sort_ok(keys[permd], rid[permd], descending=True)
    assert not checks.sort_ok(keys[permd], rid[permd])


def test_sampled_composite_key_invariants_add_up_over_shards():
    """bench.py's cfg4 gate: the invariants over the sampled composite keys
    agree with the oracle's join output, and the per-shard aggregates summed
    (the all-reduce of a multi-GPU run) equal the whole-relation ones."""
    rng = np.random.default_rng(7)
    n = 60_000
    mk = lambda: (rng.integers(0, 1 << 6, n).astype(np.int64) << np.int64(32)) | (rng.integers(0, 1 << 7, n) << 6)  # noqa
    lk, rk = mk(), mk()
    lk[::5] += 1  # keys with nonzero low bits: outside the sample (they still match each other)
    rk[::3] += 1
    lp, rp = rng.integers(-(2**40), 2**40, n), rng.integers(-(2**40), 2**40, n)
    key, lpay, rpay = O.join_columns([lk, lp], 0, [rk, rp], 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    agg = checks.sampled_join_aggregates(t(lk), t(lp), t(rk), t(rp))
    want = checks.expectations_from_aggregates(*agg)
    assert want == checks.sampled_join_observed(t(key), t(lpay), t(rpay))
    assert 0 < want["matches"] < len(key)
    h = n // 2
    a1 = checks.sampled_join_aggregates(t(lk[:h]), t(lp[:h]), t(rk[:h]), t(rp[:h]))
    a2 = checks.sampled_join_aggregates(t(lk[h:]), t(lp[h:]), t(rk[h:]), t(rp[h:]))
    assert checks.expectations_from_aggregates(*[x + y for x, y in zip(a1, a2)]) == want
