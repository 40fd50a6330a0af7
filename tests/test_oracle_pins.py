"""Pin the CPU oracle against the reference's own outputs (CPU only).

The fixtures in tests/golden/ were produced by the live reference package
(tests/golden/make_golden.py); the known answers come from the reference's
tests. Once these pass, the oracle is a trusted checker for the GPU path.
"""

import hashlib

import numpy as np
import pytest

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import synth


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sha_i64(a) -> str:
    return sha(np.asarray(a).astype("<i8"))


def test_to_tensor_small_matches_reference(golden):
    cases, arr = golden
    for i in cases["to_tensor_small"]["ids"]:
        kv, off, pos = O.to_tensor_arrays(arr[f"small{i}_keys"])
        assert kv.tolist() == arr[f"small{i}_kv"].tolist()
        assert off.tolist() == arr[f"small{i}_off"].tolist()
        assert pos.tolist() == arr[f"small{i}_pos"].tolist()


def test_to_tensor_hand_checkable():
    # test_tensorpath.py:38-47
    kv, off, pos = O.to_tensor_arrays([3, 1, 3])
    assert kv.tolist() == [1, 3]
    assert pos[off[1] : off[2]].tolist() == [0, 2]
    kv, off, pos = O.to_tensor_arrays([])
    assert len(kv) == 0 and off.tolist() == [0] and len(pos) == 0


def test_join_small_matches_reference_exact_order(golden):
    cases, arr = golden
    for i in cases["join_small"]["ids"]:
        keys, pay = arr[f"small{i}_keys"], arr[f"small{i}_pay"]
        idx = np.arange(len(keys))[::-1][: max(0, len(keys) - 3)]
        cols = O.join_columns([keys, pay], 0, [keys[idx], pay[idx]], 0)
        assert cols[0].tolist() == arr[f"join{i}_key"].tolist()
        assert (cols[1] == arr[f"join{i}_p"]).all() and (cols[2] == arr[f"join{i}_rp"]).all()


def test_join_small_matches_nested_loop(golden):
    cases, arr = golden
    for i in cases["join_small"]["ids"]:
        keys = arr[f"small{i}_keys"]
        right = keys[::-1][: max(0, len(keys) - 3)]
        l1, r1 = O.join_pairs(keys, right)
        l2, r2 = O.nested_loop_pairs(keys, right)
        assert sorted(zip(l1.tolist(), r1.tolist())) == sorted(zip(l2.tolist(), r2.tolist()))


def test_alignment_matches_reference(golden):
    _, arr = golden
    a = O.to_tensor_arrays(arr["align_a"])
    b = O.to_tensor_arrays(arr["align_b"])
    got = O.align_arrays(a[0], a[1], b[0], b[1])
    for f, g in zip(("matched_keys", "left_starts", "left_counts", "right_starts", "right_counts"), got):
        assert g.tolist() == arr[f"align_{f}"].tolist(), f
    assert got[0].tolist() == sorted(set(arr["align_a"].tolist()) & set(arr["align_b"].tolist()))


def test_generators_are_bit_exact(golden):
    cases, _ = golden
    for name, g in cases["gen"].items():
        dist = synth.Zipf(g["zipf_s"]) if g["zipf_s"] else synth.Uniform()
        rel = synth.generate_relation(synth.GenSpec(g["n"], g["domain"], dist, g["payload_width"], g["seed"]))
        assert sha_i64(rel.column("key")) == g["key_sha"], name
        assert sha(rel.column("payload")) == g["payload_sha"], name
        assert f"{O.multiset_digest(list(rel.columns)):032x}" == g["digest"], name


def test_digest_small_and_empty(golden):
    cases, arr = golden
    for i, hexd in cases["digest_small"].items():
        cols = [arr[f"small{i}_keys"], arr[f"small{i}_pay"]]
        assert f"{O.multiset_digest(cols):032x}" == hexd
    assert O.multiset_digest([np.empty(0, np.int64)]) == 0  # test_relation.py:90-93


def test_zipf_to_tensor_shas(golden):
    cases, _ = golden
    g = cases["gen"]["z100k_s6"]
    rel = synth.generate_relation(synth.GenSpec(g["n"], g["domain"], synth.Zipf(g["zipf_s"]), g["payload_width"], g["seed"]))
    kv, off, pos = O.to_tensor_arrays(rel.column("key"))
    c = cases["to_tensor_z100k"]
    assert (sha_i64(kv), sha_i64(off), sha_i64(pos)) == (c["kv_sha"], c["off_sha"], c["pos_sha"])


def test_join_20k_exact_columns_and_digest(golden):
    cases, _ = golden
    gl, gr = cases["gen"]["u20k_s16"], cases["gen"]["u20k_s17"]
    left = synth.generate_relation(synth.GenSpec(gl["n"], gl["domain"], synth.Uniform(), gl["payload_width"], gl["seed"]))
    right = synth.generate_relation(synth.GenSpec(gr["n"], gr["domain"], synth.Uniform(), gr["payload_width"], gr["seed"]))
    cols = O.join_columns(list(left.columns), 0, list(right.columns), 0)
    c = cases["join_20k"]
    assert len(cols[0]) == c["rows"]
    assert [sha(x.astype("<i8") if x.ndim == 1 else x) for x in cols] == c["col_sha"]
    assert f"{O.multiset_digest(cols):032x}" == c["digest"]


def test_cardinality_known_answer(golden):
    # test_oracles.py:22-23: 10055 for GenSpec(1000, 100, Uniform, 8, seed 21/22)
    cases, _ = golden
    gl, gr = cases["gen"]["u1000_s21"], cases["gen"]["u1000_s22"]
    lk = synth.generate_relation(synth.GenSpec(1000, 100, synth.Uniform(), 8, gl["seed"])).column("key")
    rk = synth.generate_relation(synth.GenSpec(1000, 100, synth.Uniform(), 8, gr["seed"])).column("key")
    assert O.join_count(lk, rk) == 10055 == cases["card_1000_d100"]["rows"]
    l1, r1 = O.join_pairs(lk, rk)
    l2, r2 = O.nested_loop_pairs(lk, rk)
    assert len(l1) == len(l2) == 10055
    assert O.pair_checksum(l1, r1) == O.pair_checksum(l2, r2)


@pytest.mark.slow
def test_cfg1_full_size(golden):
    c = golden[0]["cfg1"]
    r, s = synth.cfg1_relations()
    lk, rk = r.column("key"), s.column("key")
    assert O.join_count(lk, rk) == c["matches"] == 1_000_488
    kv, off, pos = O.to_tensor_arrays(lk)
    assert (len(kv), sha_i64(kv), sha_i64(off), sha_i64(pos)) == (c["d_left"], c["kv_left_sha"], c["off_left_sha"], c["pos_left_sha"])
    lrows, rrows = O.join_pairs(lk, rk)
    assert O.canonical_pairs_sha256(lrows, rrows) == c["pairs_sha"]
    assert O.pair_checksum(lrows, rrows) == c["pair_checksum"]
    cols = O.join_columns(list(r.columns), 0, list(s.columns), 0)
    assert [sha(x.astype("<i8")) for x in cols] == c["col_sha"]


@pytest.mark.slow
def test_cfg2_full_size(golden):
    c = golden[0]["cfg2"]
    rel = synth.cfg2_relation()
    keys = rel.column("key")
    assert sha_i64(keys) == c["key_input_sha"]
    perm = O.sort_permutation([keys], [False])
    assert sha_i64(perm) == c["perm_sha"]
    assert sha_i64(keys[perm]) == c["keys_sha"]
    assert sha(rel.column("payload")[perm]) == c["payload_sha"]
    assert sha_i64(O.sort_permutation([keys], [True])) == c["perm_desc_sha"]


def test_sort_three_keys(golden):
    _, arr = golden
    rng = np.random.default_rng(18)
    n = 50_000
    a = rng.integers(0, 16, n).astype(np.int64)
    b = rng.integers(-4, 4, n).astype(np.int64)
    p = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    perm = O.sort_permutation([a, p, b], [False, True, False])
    assert perm.tolist() == arr["sort3_perm"].tolist()


def test_sort_wide_bytes(golden):
    _, arr = golden
    w, k = arr["sortw_wide"], arr["sortw_k"]
    specs = {"w_asc": ([w], [False]), "w_desc": ([w], [True]), "k_desc_w_asc": ([k, w], [True, False]),
             "w_desc_k_desc": ([w, k], [True, True])}
    for tag, (cols, dirs) in specs.items():
        got = O.sort_permutation(cols, dirs)
        assert got.tolist() == arr[f"sortw_{tag}"].tolist(), tag
        small = slice(0, 300)
        assert O.sort_permutation([c[small] for c in cols], dirs).tolist() == O.comparison_sort_permutation(
            [c[small] for c in cols], dirs
        ).tolist(), tag


def test_degenerate_primary_sort():
    # test_tensorpath.py:174-186
    perm = O.sort_permutation([np.zeros(4, np.int64), np.array([2, 1, 2, 1])], [False, False])
    assert perm.tolist() == [1, 3, 0, 2]


def test_partition_hash_matches_reference(golden):
    _, arr = golden
    keys = arr["hash_keys"]
    for seed in (0, 7):
        got = O.fmix64(keys.view(np.uint64) ^ np.uint64(O.fmix64_scalar(seed)))
        assert (got == arr[f"hash_seed{seed}"]).all()


def test_chunked_pairs_concatenate_to_full():
    rng = np.random.default_rng(3)
    lk = rng.integers(0, 50, 2000)
    rk = rng.integers(0, 50, 1500)
    l_all, r_all = O.join_pairs(lk, rk)
    total = len(l_all)
    parts = [O.join_pairs(lk, rk, a, min(a + 997, total)) for a in range(0, total, 997)]
    assert np.concatenate([p[0] for p in parts]).tolist() == l_all.tolist()
    assert np.concatenate([p[1] for p in parts]).tolist() == r_all.tolist()
