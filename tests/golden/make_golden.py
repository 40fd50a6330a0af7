"""Generate the golden fixtures that pin the oracle (and, through it, the GPU).

Runs the LIVE reference package, imported read-only from
/root/reference/pkg/src, in the build container (the reference does not
exist on the GPU box, so its outputs travel as these fixtures):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden.npz (small arrays) and tests/golden/golden.json
(scalars + sha256 digests of large outputs). Each case names the reference
function that produced it.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import relab  # noqa: E402
from relab import hashing  # noqa: E402
from relab.relation import Bytes, GenSpec, Int64, Relation, Schema, Uniform, Zipf, generate_relation  # noqa: E402
from relab.specs import Direction, SortSpec  # noqa: E402
from relab.tensorpath import key_axis_align, tensor_join, tensor_sort, to_tensor  # noqa: E402

from paper_2602_21237_b200 import synth  # noqa: E402  (re-stated generators; pinned below)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sha_i64(a) -> str:
    return sha(np.asarray(a).astype("<i8"))


def to_ref(rel) -> Relation:
    """Our records.Relation → the reference Relation (same columns)."""
    attrs = tuple((n, Int64() if type(t).__name__ == "Int64" else Bytes(t.width)) for n, t in rel.schema.attributes)
    return Relation(Schema(attrs), rel.columns)


def columns_sha(rel) -> list:
    return [sha(c.astype("<i8") if c.ndim == 1 else c) for c in rel.columns]


def main() -> None:
    arrays: dict = {}
    meta: dict = {"generator": "tests/golden/make_golden.py", "reference": str(REF), "cases": {}}
    cases = meta["cases"]

    # --- small random relations with negative keys and heavy ties
    #     (the reference strategy: int64 in [-8, 8), strategies.py:27-39)
    small = []
    for i, n in enumerate([0, 1, 2, 3, 5, 17, 40, 80, 333]):
        rng = np.random.default_rng(1000 + i)
        keys = rng.integers(-8, 8, n).astype(np.int64)
        pay = rng.integers(0, 256, (n, 3), dtype=np.uint8)
        rel = Relation(Schema((("key", Int64()), ("p", Bytes(3)))), (keys, pay))
        t = to_tensor(rel, "key")
        arrays[f"small{i}_keys"] = keys
        arrays[f"small{i}_pay"] = pay
        arrays[f"small{i}_kv"] = t.key_values
        arrays[f"small{i}_off"] = t.offsets
        arrays[f"small{i}_pos"] = t.positions
        small.append(i)
    cases["to_tensor_small"] = {"ids": small, "ref": "tensorpath.py:78-93"}

    # --- joins of small relations: reversed-and-truncated self join
    #     (test_tensorpath.py:150-158) — full output columns in reference order
    for i in small:
        keys, pay = arrays[f"small{i}_keys"], arrays[f"small{i}_pay"]
        left = Relation(Schema((("key", Int64()), ("p", Bytes(3)))), (keys, pay))
        right = left.take(np.arange(left.row_count)[::-1][: max(0, left.row_count - 3)])
        out, _ = tensor_join(to_tensor(left, "key"), to_tensor(right, "key"))
        arrays[f"join{i}_key"] = out.columns[0]
        arrays[f"join{i}_p"] = out.columns[1]
        arrays[f"join{i}_rp"] = out.columns[2]
    cases["join_small"] = {"ids": small, "ref": "tensorpath.py:131-203", "right": "left reversed, last 3 dropped"}

    # --- alignment vs set oracle input (test_tensorpath.py:99-104)
    rng = np.random.default_rng(8)
    ka = rng.integers(0, 1000, 1500).astype(np.int64)
    kb = rng.integers(0, 1000, 1500).astype(np.int64)
    sch = Schema((("key", Int64()), ("p", Bytes(0))))
    al = key_axis_align(
        to_tensor(Relation(sch, (ka, np.zeros((1500, 0), np.uint8))), "key"),
        to_tensor(Relation(sch, (kb, np.zeros((1500, 0), np.uint8))), "key"),
    )
    arrays["align_a"] = ka
    arrays["align_b"] = kb
    for f in ("matched_keys", "left_starts", "left_counts", "right_starts", "right_counts"):
        arrays[f"align_{f}"] = getattr(al, f)
    cases["align_1500"] = {"ref": "tensorpath.py:109-128"}

    # --- generator pins (relation.py:283-295) for specs the tests reuse
    gens = {
        "u20k_s16": GenSpec(20_000, 500, Uniform(), 92, seed=16),
        "u20k_s17": GenSpec(20_000, 500, Uniform(), 92, seed=17),
        "z100k_s6": GenSpec(100_000, 777, Zipf(1.1), 12, seed=6),
        "u1000_s21": GenSpec(1000, 100, Uniform(), 8, seed=21),
        "u1000_s22": GenSpec(1000, 100, Uniform(), 8, seed=22),
        "z5000_s99": GenSpec(5000, 64, Zipf(1.2), 16, seed=99),
    }
    cases["gen"] = {}
    for name, g in gens.items():
        rel = generate_relation(g)
        ours = synth.generate_relation(
            synth.GenSpec(g.n, g.key_domain, synth.Zipf(g.distribution.s) if isinstance(g.distribution, Zipf)
                          else synth.Uniform(), g.payload_width, g.seed)
        )
        assert all((a == b).all() for a, b in zip(rel.columns, ours.columns)), name
        cases["gen"][name] = {
            "n": g.n, "domain": g.key_domain, "payload_width": g.payload_width, "seed": g.seed,
            "zipf_s": getattr(g.distribution, "s", None),
            "key_sha": sha_i64(rel.column("key")), "payload_sha": sha(rel.column("payload")),
            "digest": relab.multiset_digest(rel).hex,
        }

    # --- Zipf to_tensor (test_tensorpath.py:50-56)
    t = to_tensor(generate_relation(gens["z100k_s6"]), "key")
    cases["to_tensor_z100k"] = {
        "kv_sha": sha_i64(t.key_values), "off_sha": sha_i64(t.offsets), "pos_sha": sha_i64(t.positions),
        "d": int(len(t.key_values)),
    }

    # --- 20k x 20k join (test_tensorpath.py:125-130): digest + exact column order
    l20, r20 = generate_relation(gens["u20k_s16"]), generate_relation(gens["u20k_s17"])
    out, stats = tensor_join(to_tensor(l20, "key"), to_tensor(r20, "key"))
    cases["join_20k"] = {
        "rows": out.row_count, "digest": relab.multiset_digest(out).hex, "col_sha": columns_sha(out),
        "names": list(out.schema.names),
    }

    # --- cardinality known answer (test_oracles.py:22-23, 51-58)
    l1, r1 = generate_relation(gens["u1000_s21"]), generate_relation(gens["u1000_s22"])
    o1 = relab.nested_loop_join_oracle(l1, r1, "key")
    assert o1.row_count == 10055
    cases["card_1000_d100"] = {"rows": o1.row_count, "digest": relab.multiset_digest(o1).hex}

    # --- BASELINE cfg1 at full size (1M x 1M, seeds 0/1)
    r, s = synth.cfg1_relations()
    rr, ss = to_ref(r), to_ref(s)
    tr, ts = to_tensor(rr, "key"), to_tensor(ss, "key")
    out, _ = tensor_join(tr, ts)
    align = key_axis_align(tr, ts)
    lrows = out.column("payload")  # payload == row id on both sides
    rrows = out.column("right_payload")
    order = np.lexsort((rrows, lrows))
    pairs = np.stack([lrows[order], rrows[order]], axis=1).astype("<i8")
    cases["cfg1"] = {
        "matches": out.row_count, "d_left": int(len(tr.key_values)), "d_right": int(len(ts.key_values)),
        "matched_keys": int(len(align.matched_keys)),
        "max_mult_left": int(np.diff(tr.offsets).max()), "max_mult_right": int(np.diff(ts.offsets).max()),
        "pairs_sha": sha(pairs), "digest": relab.multiset_digest(out).hex, "col_sha": columns_sha(out),
        "pos_left_sha": sha_i64(tr.positions), "pos_right_sha": sha_i64(ts.positions),
        "kv_left_sha": sha_i64(tr.key_values), "off_left_sha": sha_i64(tr.offsets),
        "pair_checksum": int(
            hashing.fmix64((lrows.astype(np.uint64) << np.uint64(32)) | rrows.astype(np.uint64)).sum(dtype=np.uint64)
        ),
    }

    # --- BASELINE cfg2 at full size (10M rows, ORDER BY key)
    rel2 = synth.cfg2_relation()
    n2 = rel2.row_count
    with_id = Relation(
        Schema((("key", Int64()), ("payload", Bytes(4)), ("rid", Int64()))),
        (rel2.columns[0], rel2.columns[1], np.arange(n2, dtype=np.int64)),
    )
    out2, _ = tensor_sort(with_id, SortSpec(("key",)))
    cases["cfg2"] = {
        "n": n2, "distinct": int(len(np.unique(rel2.columns[0]))),
        "perm_sha": sha_i64(out2.column("rid")), "keys_sha": sha_i64(out2.column("key")),
        "payload_sha": sha(out2.column("payload")), "key_input_sha": sha_i64(rel2.columns[0]),
    }
    # DESC variant of the same sort (tensorpath.py:215)
    out2d, _ = tensor_sort(with_id, SortSpec(("key",), (Direction.DESC,)))
    cases["cfg2"]["perm_desc_sha"] = sha_i64(out2d.column("rid"))

    # --- 3-key sort (test_tensorpath.py:189-205) — exact permutation
    rng = np.random.default_rng(18)
    n = 50_000
    a = rng.integers(0, 16, n).astype(np.int64)
    b = rng.integers(-4, 4, n).astype(np.int64)
    p = rng.integers(0, 256, (n, 3), dtype=np.uint8)
    rel3 = Relation(
        Schema((("a", Int64()), ("b", Int64()), ("p", Bytes(3)), ("rid", Int64()))),
        (a, b, p, np.arange(n, dtype=np.int64)),
    )
    out3, _ = tensor_sort(rel3, SortSpec(("a", "p", "b"), (Direction.ASC, Direction.DESC, Direction.ASC)))
    arrays["sort3_perm"] = out3.column("rid")
    cases["sort3_50k"] = {"seed": 18, "ref": "tensorpath.py:232-252"}

    # --- wide Bytes keys (multi-word, DESC/ASC) and int64 DESC with ties
    rng = np.random.default_rng(77)
    n = 4000
    wide = rng.integers(0, 4, (n, 13), dtype=np.uint8)  # heavy ties across both words
    k64 = rng.integers(-3, 3, n).astype(np.int64)
    relw = Relation(Schema((("w", Bytes(13)), ("k", Int64()), ("rid", Int64()))), (wide, k64, np.arange(n, dtype=np.int64)))
    for tag, spec in {
        "w_asc": SortSpec(("w",)),
        "w_desc": SortSpec(("w",), (Direction.DESC,)),
        "k_desc_w_asc": SortSpec(("k", "w"), (Direction.DESC, Direction.ASC)),
        "w_desc_k_desc": SortSpec(("w", "k"), (Direction.DESC, Direction.DESC)),
    }.items():
        o, _ = tensor_sort(relw, spec)
        arrays[f"sortw_{tag}"] = o.column("rid")
    arrays["sortw_wide"] = wide
    arrays["sortw_k"] = k64
    cases["sort_wide"] = {"n": n, "seed": 77}

    # --- partition hash (hashing.py:54-61) for the multi-GPU shuffle
    rng = np.random.default_rng(5)
    hk = np.concatenate([rng.integers(-(2**62), 2**62, 1000), [0, -1, 2**63 - 1, -(2**63)]]).astype(np.int64)
    arrays["hash_keys"] = hk
    arrays["hash_seed7"] = hashing.hash_i64(hk, 7)
    arrays["hash_seed0"] = hashing.hash_i64(hk, 0)

    # --- multiset digest of assorted schemas (relation.py:319-330)
    digs = {}
    for i in small:
        keys, pay = arrays[f"small{i}_keys"], arrays[f"small{i}_pay"]
        rel = Relation(Schema((("key", Int64()), ("p", Bytes(3)))), (keys, pay))
        digs[str(i)] = relab.multiset_digest(rel).hex
    cases["digest_small"] = digs

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("wrote", HERE / "golden.npz", (HERE / "golden.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
