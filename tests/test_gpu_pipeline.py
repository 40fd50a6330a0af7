"""Device-resident pipeline (join → ORDER BY without leaving HBM), chunked
join streaming and the device digest, against the drop-in and the oracle."""

import numpy as np
import pytest
import torch

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import SortSpec, pipeline, synth, tensor_join, tensor_sort, to_tensor

pytestmark = pytest.mark.gpu


def test_join_then_order_by_equals_drop_in_and_oracle():
    n = 1_000_000
    r, s = synth.cfg1_relations(n=n, domain=n, seed=4)
    dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)
    spec = SortSpec(("payload",))
    dev_out = pipeline.join_then_order_by(dr, ds, "key", spec)
    host = dev_out.to_host()
    joined, _ = tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
    drop_in, _ = tensor_sort(joined, spec)
    assert host.schema.names == drop_in.schema.names == ("key", "payload", "right_payload")
    for a, b in zip(host.columns, drop_in.columns):
        assert (a == b).all()
    cols = O.join_columns(list(r.columns), 0, list(s.columns), 0)
    perm = O.sort_permutation([cols[1]], [False])
    for a, b in zip(host.columns, cols):
        assert (a == b[perm]).all()
    assert dev_out.digest() == O.multiset_digest(cols)


def test_join_stream_and_checksum_windows_cfg3_shape():
    r, s = synth.cfg3_relations(n=200_000)
    lk, rk = r.column("key"), s.column("key")
    plan = pipeline.plan_join(torch.from_numpy(lk.copy()).cuda(), torch.from_numpy(rk.copy()).cuda())
    assert plan.total == O.join_count(lk, rk)
    assert 5e8 < plan.total < 2e9  # the N=2e5 variant has ~9.1e8 pairs
    windows = [(0, 1 << 20), (plan.total // 3, plan.total // 3 + (1 << 20)), (plan.total - 777_777, plan.total)]
    for a, b in windows:
        got_l, got_r = [], []
        for start, lr, rr in pipeline.join_stream(plan, chunk_pairs=300_000, begin=a, end=b):
            got_l.append(lr.cpu().numpy().view(np.uint32).astype(np.int64))
            got_r.append(rr.cpu().numpy().view(np.uint32).astype(np.int64))
        wl, wr = O.join_pairs(lk, rk, a, b)
        assert (np.concatenate(got_l) == wl).all() and (np.concatenate(got_r) == wr).all()
        assert pipeline.pair_checksum(plan, a, b) == O.pair_checksum(wl, wr)


def test_order_by_multi_key_device_relation():
    rng = np.random.default_rng(6)
    n = 30_000
    from paper_2602_21237_b200 import Bytes, Direction, Int64, Relation, Schema

    rel = Relation(Schema((("a", Int64()), ("b", Bytes(5)), ("c", Int64()))),
                   (rng.integers(-3, 3, n), rng.integers(0, 3, (n, 5), dtype=np.uint8), np.arange(n)))
    spec = SortSpec(("b", "a"), (Direction.DESC, Direction.ASC))
    out, perm = pipeline.order_by(pipeline.DeviceRelation.from_host(rel), spec)
    want = O.sort_permutation([rel.column("b"), rel.column("a")], [True, False])
    assert (perm.cpu().numpy().view(np.uint32).astype(np.int64) == want).all()
    assert (out.to_host().column("c") == want).all()


def test_join_stream_vector_path_right_run_lengths():
    """Materialised pair streaming of heavy keys (4 outputs per thread,
    16-byte stores, scalar head/tail): right runs of 1, 2, 3, 7, 1023, 1025
    and 4099 rows wrap (li, ri) inside and across 4-output groups; windows
    start at odd offsets."""
    rng = np.random.default_rng(31)
    lparts, rparts = [], []
    for kv, c in zip(range(10, 17), (1, 2, 3, 7, 1023, 1025, 4099)):
        lparts.append(np.full(3000 + kv, kv, dtype=np.int64))
        rparts.append(np.full(c, kv, dtype=np.int64))
    lk = np.concatenate(lparts + [rng.integers(1000, 9000, 5000)]).astype(np.int64)
    rk = np.concatenate(rparts + [rng.integers(1000, 9000, 5000)]).astype(np.int64)
    lk, rk = lk[rng.permutation(len(lk))], rk[rng.permutation(len(rk))]
    plan = pipeline.plan_join(torch.from_numpy(lk).cuda(), torch.from_numpy(rk).cuda())
    assert plan.total == O.join_count(lk, rk)
    for a, b, chunk in ((3, plan.total, 1_000_003), (0, plan.total, 1 << 22), (plan.total // 2 + 1, plan.total, 77_777)):
        got_l, got_r = [], []
        for start, lr, rr in pipeline.join_stream(plan, chunk_pairs=chunk, begin=a, end=b):
            got_l.append(lr.cpu().numpy().view(np.uint32).astype(np.int64))
            got_r.append(rr.cpu().numpy().view(np.uint32).astype(np.int64))
        wl, wr = O.join_pairs(lk, rk, a, b)
        assert (np.concatenate(got_l) == wl).all() and (np.concatenate(got_r) == wr).all()


def test_wide_key_join_concurrent_scatter_sorts():
    """5M x 5M join on full-range int64 keys drawn from a shared pool: the join
    plan indexes both sides concurrently on half grids each, and at >= 4M wide
    keys both sorts take the scatter hybrid (chunk counts, two counting passes,
    local phase) side by side. Output byte-identical to the oracle."""
    rng = np.random.default_rng(21)
    pool = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, 3_000_000, dtype=np.int64, endpoint=True)
    n = 5_000_000
    pay = np.arange(n, dtype=np.int64)
    r = synth.Relation(synth.KEY_PAYLOAD, (pool[rng.integers(0, len(pool), n)], pay))
    s = synth.Relation(synth.KEY_PAYLOAD, (pool[rng.integers(0, len(pool), n)], pay))
    out, _ = tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
    want = O.join_columns(list(r.columns), 0, list(s.columns), 0)
    assert out.row_count == len(want[0]) > 5_000_000
    for a, b in zip(out.columns, want):
        assert (a == b).all()


@pytest.mark.parametrize("sort_col,desc", [("payload", False), ("right_payload", True), ("key", False)])
def test_fused_join_order_by_interleaved_equals_two_steps(monkeypatch, sort_col, desc):
    """join_then_order_by's fused layout (bucket join writing the two non-sort
    columns row-interleaved, one 16-byte gather a row) equals join() then
    order_by() column for column, and the oracle."""
    from paper_2602_21237_b200 import Direction

    monkeypatch.setenv("RL_FORCE_BJOIN", "1")
    n = 300_000
    r, s = synth.cfg1_relations(n=n, domain=n // 2, seed=9)
    dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)
    spec = SortSpec((sort_col,), (Direction.DESC if desc else Direction.ASC,))
    fused = pipeline.join_then_order_by(dr, ds, "key", spec).to_host()
    monkeypatch.setenv("RL_NO_FUSED_ORDER_BY", "1")
    two = pipeline.join_then_order_by(dr, ds, "key", spec).to_host()
    assert fused.schema.names == two.schema.names
    for a, b in zip(fused.columns, two.columns):
        assert a.dtype == b.dtype and (a == b).all()
    cols = O.join_columns(list(r.columns), 0, list(s.columns), 0)
    j = ("key", "payload", "right_payload").index(sort_col)
    perm = O.sort_permutation([cols[j]], [desc])
    for a, b in zip(fused.columns, cols):
        assert (a == b[perm]).all()


def test_fused_join_order_by_bytes8_payload(monkeypatch):
    """The interleaved gather moves raw 8-byte rows: a Bytes(8) payload comes
    out byte-identical to the two-step path."""
    from paper_2602_21237_b200 import records as R

    monkeypatch.setenv("RL_FORCE_BJOIN", "1")
    rng = np.random.default_rng(5)
    n = 200_000
    sch = R.Schema((("key", R.Int64()), ("payload", R.Bytes(8))))
    r = R.Relation(sch, (rng.integers(0, n, n), rng.integers(0, 256, (n, 8), dtype=np.uint8)))
    s = R.Relation(sch, (rng.integers(0, n, n), rng.integers(0, 256, (n, 8), dtype=np.uint8)))
    dr, ds = pipeline.DeviceRelation.from_host(r), pipeline.DeviceRelation.from_host(s)
    spec = SortSpec(("key",))
    fused = pipeline.join_then_order_by(dr, ds, "key", spec).to_host()
    monkeypatch.setenv("RL_NO_FUSED_ORDER_BY", "1")
    two = pipeline.join_then_order_by(dr, ds, "key", spec).to_host()
    for a, b in zip(fused.columns, two.columns):
        assert a.shape == b.shape and (a == b).all()
