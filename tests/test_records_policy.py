"""Records and path-selection policy (CPU): same behaviour as the reference's
relation/specs/selector modules (test_relation.py, test_selector.py)."""

import numpy as np
import pytest

from paper_2602_21237_b200 import (
    Bytes,
    Direction,
    GenSpec,
    Int64,
    MemoryBudget,
    Operation,
    Path,
    Policy,
    Reason,
    Relation,
    RuntimeSignals,
    Schema,
    SortSpec,
    SpillStats,
    Uniform,
    UnknownAttribute,
    estimate_intermediate,
    estimate_key_cardinality,
    generate_relation,
    join_output_schema,
    join_signals,
    select_path,
    sort_signals,
)


def signals(n_left=1000, n_right=1000, build_bytes=100_000, cardinality=1000, width=100, budget=64 * 2**20,
            op=Operation.JOIN):
    return RuntimeSignals(op, n_left, n_right, build_bytes, cardinality, width, MemoryBudget(budget))


def test_schema_rules():
    with pytest.raises(ValueError):
        Schema((("a", Int64()), ("a", Bytes(2))))
    with pytest.raises(ValueError):
        Schema(())
    s = Schema((("k", Int64()), ("p", Bytes(5)), ("q", Int64())))
    assert s.row_width == 21 and s.offsets == (0, 8, 13) and s.index("q") == 2
    with pytest.raises(UnknownAttribute):
        s.index("missing")


def test_relation_is_immutable_and_validated():
    s = Schema((("k", Int64()), ("p", Bytes(3))))
    with pytest.raises(ValueError):
        Relation(s, (np.zeros(2, np.int64), np.zeros((3, 3), np.uint8)))
    rel = Relation(s, (np.arange(3), np.zeros((3, 3), np.uint8)))
    assert not rel.column("k").flags.writeable
    assert rel.take([2, 0]).column("k").tolist() == [2, 0]
    assert Relation.from_rows(s, rel.row_tuples()).row_tuples() == rel.row_tuples()
    assert rel.serialize().shape == (3, 11)


def test_join_output_schema_collisions():
    s = Schema((("key", Int64()), ("v", Bytes(1))))
    out = join_output_schema(s, s, "key")
    assert out.names == ("key", "v", "right_v")
    with pytest.raises(UnknownAttribute):
        join_output_schema(Schema((("key", Bytes(8)),)), s, "key")


def test_sort_spec_defaults_and_errors():
    assert SortSpec(("a", "b")).directions == (Direction.ASC, Direction.ASC)
    assert SortSpec(("a",), ("desc",)).directions == (Direction.DESC,)
    with pytest.raises(ValueError):
        SortSpec(())
    with pytest.raises(ValueError):
        SortSpec(("a", "a"))
    with pytest.raises(ValueError):
        MemoryBudget(1024)


def test_spill_stats_zero_and_mb():
    s = SpillStats()
    assert s.temp_mb == 0.0 and s.copy() == s
    assert SpillStats(temp_blocks_written=128).temp_mb == 1.0


def test_estimates():
    assert estimate_intermediate(signals(n_left=0, n_right=0, cardinality=0)) == 0
    assert estimate_intermediate(signals(200, 300, cardinality=1, width=10)) == 200 * 300 * 10
    assert estimate_intermediate(signals(500, width=24, op=Operation.SORT)) == 500 * 24


def test_select_rules_and_boundary():
    assert select_path(signals(build_bytes=10 * 2**20)).reason is Reason.FITS_IN_MEMORY
    c = select_path(signals(1_000_000, 1_000_000, 100 * 2**20, budget=2**20))
    assert (c.path, c.reason) == (Path.TENSOR, Reason.SPILL_RISK_HIGH)
    c = select_path(signals(10_000, 10_000, 2 * 2**20, budget=2**20))
    assert (c.path, c.reason) == (Path.ROW, Reason.SMALL_INPUT)
    assert select_path(signals(), Policy.FORCE_TENSOR).path is Path.TENSOR
    assert select_path(signals(), Policy.FORCE_ROW).reason is Reason.FORCED
    at = signals(build_bytes=int(0.75 * 2**20), budget=2**20)
    over = signals(60_000, 60_000, int(0.75 * 2**20) + 1, budget=2**20)
    assert select_path(at).reason is Reason.FITS_IN_MEMORY
    assert select_path(over).reason is Reason.SPILL_RISK_HIGH
    assert len({select_path(at) for _ in range(100)}) == 1
    with pytest.raises(ValueError):
        signals(n_left=-1)


def test_baseline_sweep_sizes_choose_tensor():
    """BASELINE cfg5: at work_mem = 1 MB every N in 1e5..1e9 selects TENSOR."""
    for n in (10**5, 10**6, 10**7, 10**8, 10**9):
        s = RuntimeSignals(Operation.JOIN, n, n, n * 16, n, 24, MemoryBudget(2**20))
        assert select_path(s).path is Path.TENSOR
        s = RuntimeSignals(Operation.SORT, n, 0, n * 24, 0, 24, MemoryBudget(2**20))
        assert select_path(s).path is Path.TENSOR


def test_key_cardinality_and_signal_builders():
    rel = generate_relation(GenSpec(2000, 64, Uniform(), 0, seed=2))
    assert estimate_key_cardinality(rel, "key") == len(np.unique(rel.column("key")))
    big = generate_relation(GenSpec(100_000, 5000, Uniform(), 0, seed=3))
    truth = len(np.unique(big.column("key")))
    assert truth / 3 <= estimate_key_cardinality(big, "key") <= truth * 3
    left = generate_relation(GenSpec(1000, 50, Uniform(), 12, seed=1))
    right = generate_relation(GenSpec(500, 50, Uniform(), 12, seed=2))
    s = join_signals(left, right, "key", MemoryBudget(2**20))
    assert s.serialized_bytes_build == 500 * 20 and s.output_row_width == 32
    assert s.expected_intermediate_bytes == estimate_intermediate(s)
    ss = sort_signals(left, MemoryBudget(2**20))
    assert ss.operation is Operation.SORT and ss.serialized_bytes_build == 1000 * 20
