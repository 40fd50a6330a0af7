"""The restated CPU relational baseline (oracle/relational_baseline.py) —
bench.py's reference-path timing — pinned against the live reference's
rowpath.hash_join_row (temp blocks, partition passes, match count) where
/root/reference exists, and against the SURVEY's measured cfg1 figures."""

from pathlib import Path

import numpy as np
import pytest

from oracle import relational_baseline as RB
from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import synth

REF = Path("/root/reference/pkg/src")


def test_cfg1_spill_counts_match_survey():
    """SURVEY §6 (its probe used seeds 1/2): cfg1 at work_mem = 1 MB joins
    999,411 rows and spills 3,933 blocks (30.73 MB) in one partition pass;
    the bench's seeds 0/1 spill 3,931 blocks for 1,000,488 rows."""
    for seed, rows_want, blocks in ((1, 999_411, 3933), (0, 1_000_488, 3931)):
        r, s = synth.cfg1_relations(seed=seed)
        rows, st = RB.hash_join_row(list(r.columns), [8, 8], 0, list(s.columns), [8, 8], 0, 1 << 20)
        assert rows == rows_want == O.join_count(r.column("key"), s.column("key"))
        assert st.temp_blocks_written == blocks and st.partition_passes == 1
    assert round(3933 * RB.BLOCK_SIZE / 2**20, 2) == 30.73


@pytest.mark.skipif(not REF.exists(), reason="the reference package is only in the build container")
@pytest.mark.parametrize("n,dom,width,budget", [(60_000, 20_000, 8, 65536), (200_000, 500, 20, 1 << 20),
                                                (30_000, 30_000, 0, 65536)])
def test_against_live_reference(tmp_path, n, dom, width, budget):
    import sys

    sys.path.insert(0, str(REF))
    from relab import relation as rel
    from relab.rowpath import hash_join_row
    from relab.specs import JoinSpec, MemoryBudget
    from relab.spill import TempArena

    rng = np.random.default_rng(n + dom)
    cols = []
    for _ in range(2):
        k = rng.integers(-dom, dom, n).astype(np.int64)
        p = rng.integers(0, 256, (n, width), dtype=np.uint8)
        cols.append((k, p))
    schema = rel.Schema((("key", rel.Int64()), ("p", rel.Bytes(width))))
    L, R_ = (rel.Relation(schema, c) for c in cols)
    with TempArena(tmp_path) as arena:
        out, st = hash_join_row(L, R_, JoinSpec("key"), MemoryBudget(budget), arena)
    rows, mine = RB.hash_join_row(list(cols[0]), [8, width], 0, list(cols[1]), [8, width], 0, budget, tmp_path)
    assert rows == out.row_count
    assert mine.temp_blocks_written == st.temp_blocks_written
    assert mine.temp_bytes_written == st.temp_bytes_written
    assert mine.partition_passes == st.partition_passes
