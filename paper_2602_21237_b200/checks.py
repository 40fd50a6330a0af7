"""Size-independent result checks for joins and sorts too large for the CPU
oracle (BASELINE cfg5 at 1e8-1e9 rows, the north star's 1B-row join).

Everything here is computed with stock torch ops (bincount, scatter_add,
sort) on the INPUTS, independently of librelab_b200.so, and compared with
the same quantities read off the library's OUTPUT. They back the bench's
correctness gates and the large-size GPU tests; at the sizes the oracle
finishes in seconds, the tests compare full columns with the oracle instead.

For an equi-join of L(key, lpay) with R(key, rpay), with c_L(k), c_R(k) the
key multiplicities and S_L(k) = sum of f(lpay) over left rows with key k:

* matches            = sum_k c_L(k) c_R(k)               (test_oracles.py:55-57)
* sum of out keys    = sum_k k c_L(k) c_R(k)
* sum of f(lpay)     = sum_k S_L(k) c_R(k),  likewise for the right side
* sum f(lpay) g(rpay) = sum_k S_L(k) S_R(k)   (pairs the right rows with the
  right left rows, not just the right multisets)

all in wrapping int64 arithmetic (mod 2^64) on both sides. The order checks
follow tensorpath.py:162-172 (key, left row, right row) and the stable
ORDER BY of tensorpath.py:232-252.
"""

from __future__ import annotations

import torch

_F = -7046029254386353131  # 0x9E3779B97F4A7C15 as int64 (odd: a bijection mod 2^64)
_G = -4658895280553007687  # 0xBF58476D1CE4E5B9 as int64


def _f(x: torch.Tensor) -> torch.Tensor:
    return x * _F + 0x632BE59BD9B4E019


def _g(x: torch.Tensor) -> torch.Tensor:
    return (x ^ 0x94D049BB133111EB) * _G


FIELDS = ("matches", "sum_key", "sum_f_left", "sum_g_right", "sum_pair")


def join_aggregates(lk, lpay, rk, rpay, domain: int):
    """Per-key aggregates of keys in [0, domain): (c_L, c_R, S_L, S_R). They add
    up over row shards, so ranks holding parts of L and R all-reduce them."""
    cl = torch.bincount(lk, minlength=domain)
    cr = torch.bincount(rk, minlength=domain)
    sl = torch.zeros(domain, dtype=torch.int64, device=lk.device).scatter_add_(0, lk, _f(lpay))
    sr = torch.zeros(domain, dtype=torch.int64, device=lk.device).scatter_add_(0, rk, _g(rpay))
    return cl, cr, sl, sr


def expectations_from_aggregates(cl, cr, sl, sr, keyval=None) -> dict:
    if keyval is None:
        keyval = torch.arange(cl.numel(), device=cl.device, dtype=torch.int64)
    return {
        "matches": int((cl * cr).sum()),
        "sum_key": int((keyval * cl * cr).sum()),
        "sum_f_left": int((sl * cr).sum()),
        "sum_g_right": int((sr * cl).sum()),
        "sum_pair": int((sl * sr).sum()),
    }


def join_expectations(lk, lpay, rk, rpay, domain=None) -> dict:
    """The invariants above from the inputs (device int64 tensors). Keys in
    [0, domain) are their own dense ids; otherwise torch.unique ranks them."""
    if domain is not None:
        return expectations_from_aggregates(*join_aggregates(lk, lpay, rk, rpay, int(domain)))
    uniq, inv = torch.unique(torch.cat([lk, rk]), return_inverse=True)
    agg = join_aggregates(inv[: lk.numel()], lpay, inv[lk.numel():], rpay, uniq.numel())
    return expectations_from_aggregates(*agg, keyval=uniq)


def join_observed(out_key, out_lpay, out_rpay) -> dict:
    """The same quantities read off a join's output columns."""
    return {
        "matches": int(out_key.numel()),
        "sum_key": int(out_key.sum()),
        "sum_f_left": int(_f(out_lpay).sum()),
        "sum_g_right": int(_g(out_rpay).sum()),
        "sum_pair": int((_f(out_lpay) * _g(out_rpay)).sum()),
    }


def join_order_ok(out_key, out_lrow, out_rrow) -> bool:
    """Output rows in the reference order: key ascending, then left row,
    then right row (tensorpath.py:162-172; left/right rows = the payloads
    when the payload is the row id)."""
    if out_key.numel() < 2:
        return True
    k0, k1 = out_key[:-1], out_key[1:]
    l0, l1 = out_lrow[:-1], out_lrow[1:]
    r0, r1 = out_rrow[:-1], out_rrow[1:]
    ok = (k0 < k1) | ((k0 == k1) & ((l0 < l1) | ((l0 == l1) & (r0 < r1))))
    return bool(ok.all())


def sort_ok(sorted_key, tie_col=None, descending: bool = False) -> bool:
    """Sorted by the key; where keys tie, `tie_col` (the rows' previous
    order, e.g. a row id carried along) ascends: the stable order."""
    if sorted_key.numel() < 2:
        return True
    a, b = sorted_key[:-1], sorted_key[1:]
    ok = (a >= b) if descending else (a <= b)
    if tie_col is not None:
        ok = ok & ((a != b) | (tie_col[:-1] < tie_col[1:]))
    return bool(ok.all())


def multiset_sums(cols) -> tuple:
    """Order-independent sums of a relation's int64 columns (a permutation of
    the rows leaves them unchanged): per column sum f(x), plus the sum of
    f(first) g(second) tying the first two columns together row by row."""
    out = [int(_f(c).sum()) for c in cols]
    if len(cols) > 1:
        out.append(int((_f(cols[0]) * _g(cols[1])).sum()))
    return tuple(out)


def sampled_join_aggregates(lk, lpay, rk, rpay, sample_bits: int = 6, id_bits: int = 26):
    """join_aggregates over the keys whose low `sample_bits` bits are zero
    (1 in 2^sample_bits of a uniform key space), keyed by a dense id: for
    composite keys (a << 32) | b with a, b < 2^16 (BASELINE cfg4) the id is
    (a << (16 - sample_bits)) | (b >> sample_bits). Bounded memory whatever
    the key space; the aggregates still add up over row shards."""
    def ids(k):
        a, b = k >> 32, k & 0xFFFF
        keep = (k & ((1 << sample_bits) - 1)) == 0
        return keep, (a << (16 - sample_bits)) | (b >> sample_bits)

    dom = 1 << id_bits
    kl, il = ids(lk)
    kr, ir = ids(rk)
    return join_aggregates(il[kl], lpay[kl], ir[kr], rpay[kr], dom)


def sampled_join_observed(out_key, out_lpay, out_rpay, sample_bits: int = 6) -> dict:
    keep = (out_key & ((1 << sample_bits) - 1)) == 0
    k = out_key[keep]
    a, b = k >> 32, k & 0xFFFF
    dense = (a << (16 - sample_bits)) | (b >> sample_bits)
    return join_observed(dense, out_lpay[keep], out_rpay[keep])
