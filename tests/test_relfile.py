"""RELCOL01 relation files (relation.py:364-419): the header codec here (CPU)
and the device / page-locked readers and the device writer (GPU), checked
against a restatement of the reference's writer and reader."""

import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2602_21237_b200 import records as R
from paper_2602_21237_b200 import relfile


def ref_write(path, names_types, cols, n):
    """Restatement of relation.py:379-392 (write_relation) for the tests."""
    attrs = [[nm, "int64" if t == "int64" else ["bytes", t]] for nm, t in names_types]
    header = json.dumps({"attrs": attrs, "rows": n}).encode()
    with open(path, "wb") as f:
        f.write(b"RELCOL01")
        f.write(len(header).to_bytes(4, "little"))
        f.write(header)
        for c, (_, t) in zip(cols, names_types):
            f.write(c.astype("<i8").tobytes() if t == "int64" else c.tobytes())


def sample(n, seed=0):
    rng = np.random.default_rng(seed)
    nt = [("key", "int64"), ("pay", 5), ("empty", 0), ("v", "int64")]
    cols = [rng.integers(-(2**63), 2**63 - 1, n, dtype=np.int64, endpoint=True),
            rng.integers(0, 256, (n, 5), dtype=np.uint8), np.zeros((n, 0), dtype=np.uint8),
            np.arange(n, dtype=np.int64)]
    return nt, cols


def schema_of(nt):
    return R.Schema(tuple((nm, R.Int64() if t == "int64" else R.Bytes(t)) for nm, t in nt))


def test_header_codec_matches_reference(tmp_path):
    nt, cols = sample(1000)
    p = tmp_path / "r.relcol"
    ref_write(p, nt, cols, 1000)
    head = relfile.header_bytes(schema_of(nt), 1000)
    assert p.read_bytes()[:len(head)] == head
    schema, n, sections = relfile.read_header(p)
    assert n == 1000 and [a for a, _ in schema.attributes] == ["key", "pay", "empty", "v"]
    assert [w for _, w in sections] == [8, 5, 0, 8]
    assert sections[0][0] == len(head) and sections[1][0] == len(head) + 8000


def test_header_errors(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTAFILE" + b"\0" * 8)
    with pytest.raises(ValueError, match="not a relation file"):
        relfile.read_header(bad)
    nt, cols = sample(100)
    p = tmp_path / "t"
    ref_write(p, nt, cols, 100)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(ValueError, match="truncated"):
        relfile.read_header(p)


@pytest.mark.skipif(not Path("/root/reference/pkg/src/relab/relation.py").exists(),
                    reason="the reference package is only in the build container")
def test_header_codec_against_live_reference(tmp_path):
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from relab import relation as ref

    nt, cols = sample(300, 3)
    rel = ref.Relation(ref.Schema(tuple((nm, ref.Int64() if t == "int64" else ref.Bytes(t)) for nm, t in nt)),
                       tuple(cols))
    p = tmp_path / "live"
    ref.write_relation(rel, p)
    mine = tmp_path / "mine"
    ref_write(mine, nt, cols, 300)
    assert p.read_bytes() == mine.read_bytes()


@pytest.mark.gpu
def test_device_round_trip_and_reference_bytes(tmp_path):
    from paper_2602_21237_b200 import _capi, pipeline

    n = 3_000_001  # several 8 MiB staging chunks, ragged
    nt, cols = sample(n, 1)
    ref_path = tmp_path / "ref"
    ref_write(ref_path, nt, cols, n)
    dr = pipeline.DeviceRelation.from_file(ref_path)
    for got, want in zip(dr.columns, cols):
        assert (got.cpu().numpy() == want).all()
    out = tmp_path / "out"
    dr.to_file(out)
    assert out.read_bytes() == ref_path.read_bytes()
    shard = pipeline.DeviceRelation.from_file(ref_path, rows=(1_234_567, 2_000_003))
    for got, want in zip(shard.columns, cols):
        assert (got.cpu().numpy() == want[1_234_567:2_000_003]).all()
    rel = relfile.read_pinned(ref_path)
    lib = _capi.load()
    for got, want in zip(rel.columns, cols):
        assert (got == want).all()
    assert lib.rl_host_is_pinned(rel.columns[0].ctypes.data) == 1
    with pytest.raises(ValueError):
        pipeline.DeviceRelation.from_file(ref_path, rows=(5, n + 1))
