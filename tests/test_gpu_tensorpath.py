"""GPU parity of the drop-in operators — the reference's test_tensorpath.py
(/root/reference/pkg/tests/test_tensorpath.py) restated against the B200
implementation, with the pinned CPU oracle as the checker, plus bit-exact
comparisons against the reference's golden outputs."""

import hashlib

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import (
    Bytes,
    Direction,
    GenSpec,
    Int64,
    OutputTooLarge,
    Relation,
    Schema,
    SortSpec,
    Uniform,
    UnknownAttribute,
    Zipf,
    generate_relation,
    key_axis_align,
    tensor_join,
    tensor_sort,
    to_tensor,
)

pytestmark = pytest.mark.gpu


def digest(rel) -> int:
    return O.multiset_digest(list(rel.columns))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@st.composite
def relations(draw, max_rows=80, key_range=8):
    """The reference strategy (strategies.py:14-39): an int64 'key' plus up to
    two extra Int64/Bytes(0..6) columns, values in [-8, 8)."""
    attrs = [("key", Int64())]
    for i in range(draw(st.integers(0, 2))):
        attrs.append((f"c{i}", Int64() if draw(st.booleans()) else Bytes(draw(st.integers(0, 6)))))
    schema = Schema(tuple(attrs))
    n = draw(st.integers(0, max_rows))
    rng = np.random.default_rng(draw(st.integers(0, 2**32 - 1)))
    cols = [
        rng.integers(-key_range, key_range, n).astype(np.int64) if isinstance(t, Int64)
        else rng.integers(0, 256, (n, t.width), dtype=np.uint8)
        for _, t in schema.attributes
    ]
    return Relation(schema, tuple(cols))


# ------------------------------------------------------------------ to_tensor
def test_to_tensor_empty():
    t = to_tensor(generate_relation(GenSpec(0, 1, Uniform(), 4, seed=0)), "key")
    assert len(t.key_values) == 0
    assert t.offsets.tolist() == [0]
    assert t.row_count == 0


def test_to_tensor_hand_checkable_stability():
    schema = Schema((("key", Int64()), ("p", Bytes(0))))
    rel = Relation(schema, (np.array([3, 1, 3], dtype=np.int64), np.zeros((3, 0), dtype=np.uint8)))
    t = to_tensor(rel, "key")
    assert t.key_values.tolist() == [1, 3]
    assert t.positions[t.offsets[1] : t.offsets[2]].tolist() == [0, 2]
    assert t.positions.dtype == np.int64 and t.offsets.dtype == np.int64


def test_to_tensor_round_trip_and_zipf_golden(golden):
    cases, _ = golden
    rel = generate_relation(GenSpec(100_000, 777, Zipf(1.1), 12, seed=6))
    t = to_tensor(rel, "key")
    assert digest(t.to_relation()) == digest(rel)
    assert np.sort(t.positions).tolist() == list(range(rel.row_count))
    c = cases["to_tensor_z100k"]
    assert sha(t.key_values.astype("<i8")) == c["kv_sha"]
    assert sha(t.offsets.astype("<i8")) == c["off_sha"]
    assert sha(t.positions.astype("<i8")) == c["pos_sha"]


def test_to_tensor_requires_int64_key():
    rel = generate_relation(GenSpec(5, 2, Uniform(), 4, seed=1))
    with pytest.raises(UnknownAttribute):
        to_tensor(rel, "payload")
    with pytest.raises(UnknownAttribute):
        to_tensor(rel, "nope")


def test_to_tensor_small_golden_bit_exact(golden):
    cases, arr = golden
    for i in cases["to_tensor_small"]["ids"]:
        rel = Relation(Schema((("key", Int64()), ("p", Bytes(3)))), (arr[f"small{i}_keys"], arr[f"small{i}_pay"]))
        t = to_tensor(rel, "key")
        assert t.key_values.tolist() == arr[f"small{i}_kv"].tolist()
        assert t.offsets.tolist() == arr[f"small{i}_off"].tolist()
        assert t.positions.tolist() == arr[f"small{i}_pos"].tolist()


@given(relations(max_rows=60))
def test_to_tensor_invariants(rel):
    t = to_tensor(rel, "key")
    kv, off, pos = O.to_tensor_arrays(rel.column("key"))
    assert t.key_values.tolist() == kv.tolist()
    assert t.offsets.tolist() == off.tolist()
    assert t.positions.tolist() == pos.tolist()


def test_to_tensor_extreme_keys():
    keys = np.array([2**63 - 1, -(2**63), 0, -1, 1, 2**63 - 1, -(2**63), 5], dtype=np.int64)
    rel = Relation(Schema((("key", Int64()),)), (keys,))
    t = to_tensor(rel, "key")
    kv, off, pos = O.to_tensor_arrays(keys)
    assert (t.key_values.tolist(), t.offsets.tolist(), t.positions.tolist()) == (kv.tolist(), off.tolist(), pos.tolist())


def _tensor_from_keys(keys):
    schema = Schema((("key", Int64()), ("p", Bytes(0))))
    keys = np.asarray(keys, dtype=np.int64)
    return to_tensor(Relation(schema, (keys, np.zeros((len(keys), 0), dtype=np.uint8))), "key")


# ------------------------------------------------------------------ alignment
def test_alignment_simple_and_disjoint():
    assert key_axis_align(_tensor_from_keys([1, 2, 3]), _tensor_from_keys([2, 3, 4])).matched_keys.tolist() == [2, 3]
    assert len(key_axis_align(_tensor_from_keys([1, 2]), _tensor_from_keys([5, 9])).matched_keys) == 0
    assert len(key_axis_align(_tensor_from_keys([]), _tensor_from_keys([5, 9])).matched_keys) == 0
    assert len(key_axis_align(_tensor_from_keys([1]), _tensor_from_keys([])).matched_keys) == 0


def test_alignment_matches_reference_golden(golden):
    _, arr = golden
    al = key_axis_align(_tensor_from_keys(arr["align_a"]), _tensor_from_keys(arr["align_b"]))
    for f in ("matched_keys", "left_starts", "left_counts", "right_starts", "right_counts"):
        assert getattr(al, f).tolist() == arr[f"align_{f}"].tolist(), f
    assert al.matched_keys.tolist() == sorted(set(arr["align_a"].tolist()) & set(arr["align_b"].tolist()))


# ------------------------------------------------------------------ join
def test_tensor_join_trivial_example():
    schema = Schema((("key", Int64()), ("v", Bytes(1))))
    left = Relation.from_rows(schema, [(1, b"a")])
    right = Relation.from_rows(schema, [(1, b"x"), (2, b"y")])
    out, stats = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))
    assert out.row_tuples() == [(1, b"a", b"x")]
    assert out.schema.names == ("key", "v", "right_v")
    assert stats.temp_blocks_written == 0


def test_tensor_join_zero_spill_structural():
    left = generate_relation(GenSpec(5000, 100, Uniform(), 16, seed=1))
    right = generate_relation(GenSpec(5000, 100, Uniform(), 16, seed=2))
    _, stats = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))
    assert stats.temp_blocks_written == stats.temp_bytes_written == stats.temp_bytes_read == 0


def test_tensor_join_20k_bit_exact_vs_reference(golden):
    c = golden[0]["join_20k"]
    left = generate_relation(GenSpec(20_000, 500, Uniform(), 92, seed=16))
    right = generate_relation(GenSpec(20_000, 500, Uniform(), 92, seed=17))
    out, _ = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))
    assert out.row_count == c["rows"]
    assert list(out.schema.names) == c["names"]
    assert [sha(x.astype("<i8") if x.ndim == 1 else x) for x in out.columns] == c["col_sha"]
    assert f"{digest(out):032x}" == c["digest"]


def test_tensor_join_small_golden_exact_order(golden):
    cases, arr = golden
    for i in cases["join_small"]["ids"]:
        schema = Schema((("key", Int64()), ("p", Bytes(3))))
        left = Relation(schema, (arr[f"small{i}_keys"], arr[f"small{i}_pay"]))
        right = left.take(np.arange(left.row_count)[::-1][: max(0, left.row_count - 3)])
        out, _ = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))
        assert out.column("key").tolist() == arr[f"join{i}_key"].tolist()
        assert (out.column("p") == arr[f"join{i}_p"]).all()
        assert (out.column("right_p") == arr[f"join{i}_rp"]).all()


def test_tensor_join_output_cap():
    left = generate_relation(GenSpec(3000, 1, Uniform(), 0, seed=1))
    right = generate_relation(GenSpec(3000, 1, Uniform(), 0, seed=2))
    with pytest.raises(OutputTooLarge):
        tensor_join(to_tensor(left, "key"), to_tensor(right, "key"), max_output_rows=10_000)
    out, _ = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"), max_output_rows=9_000_000)
    assert out.row_count == 9_000_000


def test_tensor_join_different_keys_rejected():
    s = Schema((("key", Int64()), ("k2", Int64())))
    rel = Relation(s, (np.arange(3), np.arange(3)))
    with pytest.raises(UnknownAttribute):
        tensor_join(to_tensor(rel, "key"), to_tensor(rel, "k2"))


def test_tensor_join_memory_accounting_deterministic():
    left = generate_relation(GenSpec(10_000, 200, Uniform(), 24, seed=3))
    right = generate_relation(GenSpec(10_000, 200, Uniform(), 24, seed=4))
    peaks = {tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))[1].peak_mem_bytes for _ in range(3)}
    assert len(peaks) == 1 and peaks.pop() > 0


@given(relations(max_rows=50))
def test_tensor_join_matches_oracle_property(left):
    right = left.take(np.arange(left.row_count)[::-1][: max(0, left.row_count - 3)])
    out, stats = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))
    assert stats.temp_blocks_written == 0
    k = left.schema.index("key")
    want = O.join_columns(list(left.columns), k, list(right.columns), k)
    assert len(out.columns) == len(want)
    for got, exp in zip(out.columns, want):  # byte-identical, same row order
        assert got.shape == exp.shape and (got == exp).all()


@given(relations(max_rows=70), relations(max_rows=70))
def test_tensor_join_two_relations_vs_nested_loop(left, right):
    lt, rt = to_tensor(left, "key"), to_tensor(right, "key")
    out, _ = tensor_join(lt, rt)
    l2, r2 = O.nested_loop_pairs(left.column("key"), right.column("key"))
    assert out.row_count == len(l2)
    if len(l2):
        kk = right.schema.index("key")
        want = [c[l2] for c in left.columns] + [c[r2] for j, c in enumerate(right.columns) if j != kk]
        assert O.multiset_digest(list(out.columns)) == O.multiset_digest(want)


def test_tensor_join_accepts_host_built_tensor_relation():
    from paper_2602_21237_b200 import TensorRelation

    rel = generate_relation(GenSpec(500, 40, Uniform(), 4, seed=9))
    kv, off, pos = O.to_tensor_arrays(rel.column("key"))
    host_built = TensorRelation(rel.schema, rel.columns, "key", kv, off, pos)
    out, _ = tensor_join(host_built, to_tensor(rel, "key"))
    want = O.join_columns(list(rel.columns), 0, list(rel.columns), 0)
    assert all((a == b).all() for a, b in zip(out.columns, want))
    with pytest.raises(ValueError):
        TensorRelation(rel.schema, rel.columns, "key", kv[::-1], off, pos)


# ------------------------------------------------------------------ sort
def test_tensor_sort_single_key():
    schema = Schema((("key", Int64()), ("p", Bytes(0))))
    rel = Relation(schema, (np.array([2, 1], dtype=np.int64), np.zeros((2, 0), dtype=np.uint8)))
    out, stats = tensor_sort(rel, SortSpec(("key",)))
    assert out.column("key").tolist() == [1, 2]
    assert stats.temp_blocks_written == 0


def test_tensor_sort_degenerate_primary():
    schema = Schema((("a", Int64()), ("b", Int64()), ("tag", Int64())))
    rel = Relation(schema, (np.zeros(4, np.int64), np.array([2, 1, 2, 1], np.int64), np.arange(4, dtype=np.int64)))
    out, _ = tensor_sort(rel, SortSpec(("a", "b")))
    assert out.column("tag").tolist() == [1, 3, 0, 2]


def test_tensor_sort_three_keys_matches_reference_50k(golden):
    _, arr = golden
    rng = np.random.default_rng(18)
    n = 50_000
    schema = Schema((("a", Int64()), ("b", Int64()), ("p", Bytes(3)), ("rid", Int64())))
    rel = Relation(schema, (rng.integers(0, 16, n).astype(np.int64), rng.integers(-4, 4, n).astype(np.int64),
                            rng.integers(0, 256, (n, 3), dtype=np.uint8), np.arange(n, dtype=np.int64)))
    out, stats = tensor_sort(rel, SortSpec(("a", "p", "b"), (Direction.ASC, Direction.DESC, Direction.ASC)))
    assert stats.temp_blocks_written == 0
    assert out.column("rid").tolist() == arr["sort3_perm"].tolist()
    want = rel.take(arr["sort3_perm"])
    assert all((x == y).all() for x, y in zip(out.columns, want.columns))


def test_tensor_sort_wide_bytes_golden(golden):
    _, arr = golden
    w, k = arr["sortw_wide"], arr["sortw_k"]
    n = len(k)
    rel = Relation(Schema((("w", Bytes(13)), ("k", Int64()), ("rid", Int64()))), (w, k, np.arange(n, dtype=np.int64)))
    specs = {"w_asc": SortSpec(("w",)), "w_desc": SortSpec(("w",), (Direction.DESC,)),
             "k_desc_w_asc": SortSpec(("k", "w"), (Direction.DESC, Direction.ASC)),
             "w_desc_k_desc": SortSpec(("w", "k"), (Direction.DESC, Direction.DESC))}
    for tag, spec in specs.items():
        out, _ = tensor_sort(rel, spec)
        assert out.column("rid").tolist() == arr[f"sortw_{tag}"].tolist(), tag


@given(relations(max_rows=60))
def test_tensor_sort_radix_identity_property(rel):
    keys = list(rel.schema.names)
    dirs = [Direction.DESC if i % 2 else Direction.ASC for i in range(len(keys))]
    out, _ = tensor_sort(rel, SortSpec(tuple(keys), tuple(dirs)))
    perm = O.comparison_sort_permutation(list(rel.columns), [d is Direction.DESC for d in dirs])
    want = rel.take(perm)
    assert out.row_tuples() == want.row_tuples()


def test_tensor_sort_unknown_key_and_empty():
    rel = Relation(Schema((("key", Int64()),)), (np.array([3, 1], np.int64),))
    with pytest.raises(UnknownAttribute):
        tensor_sort(rel, SortSpec(("nope",)))
    empty = Relation(Schema((("key", Int64()),)), (np.empty(0, np.int64),))
    out, stats = tensor_sort(empty, SortSpec(("key",)))
    assert out.row_count == 0 and stats.temp_blocks_written == 0


def test_tensor_sort_extreme_int64_desc():
    keys = np.array([0, -1, 2**63 - 1, -(2**63), 7, -(2**63), 2**63 - 1, 0], dtype=np.int64)
    rel = Relation(Schema((("key", Int64()), ("rid", Int64()))), (keys, np.arange(len(keys), dtype=np.int64)))
    for desc in (False, True):
        out, _ = tensor_sort(rel, SortSpec(("key",), (Direction.DESC if desc else Direction.ASC,)))
        assert out.column("rid").tolist() == O.comparison_sort_permutation([keys], [desc]).tolist()
