"""Device multiset digest == the reference's (golden) and the oracle's."""

import numpy as np
import pytest
import torch

from oracle import tensorpath_oracle as O
from paper_2602_21237_b200 import engine, synth, tensor_join, to_tensor
from paper_2602_21237_b200.tensor_path import multiset_digest

pytestmark = pytest.mark.gpu


def test_digest_matches_reference_goldens(golden):
    cases, arr = golden
    for i, hexd in cases["digest_small"].items():
        cols = [torch.from_numpy(arr[f"small{i}_keys"]).cuda(), torch.from_numpy(arr[f"small{i}_pay"]).cuda()]
        assert f"{engine.multiset_digest(cols):032x}" == hexd
    for name, g in cases["gen"].items():
        dist = synth.Zipf(g["zipf_s"]) if g["zipf_s"] else synth.Uniform()
        rel = synth.generate_relation(synth.GenSpec(g["n"], g["domain"], dist, g["payload_width"], g["seed"]))
        assert f"{multiset_digest(rel):032x}" == g["digest"], name


def test_digest_of_cfg1_join_output_on_device(golden):
    r, s = synth.cfg1_relations()
    out, _ = tensor_join(to_tensor(r, "key"), to_tensor(s, "key"))
    assert f"{multiset_digest(out):032x}" == golden[0]["cfg1"]["digest"]


@pytest.mark.parametrize("widths", [(8,), (8, 0), (8, 3, 8), (1, 2, 5, 8, 13), (8, 92), (8, 8, 8)])
def test_digest_matches_oracle_any_layout(widths):
    rng = np.random.default_rng(sum(widths))
    n = 3001
    cols = [rng.integers(-(2**62), 2**62, n) if w == 8 and j % 2 == 0 else rng.integers(0, 256, (n, w), dtype=np.uint8)
            for j, w in enumerate(widths)]
    got = engine.multiset_digest([torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols])
    assert got == O.multiset_digest(cols)
    assert engine.multiset_digest([torch.empty(0, dtype=torch.int64, device="cuda")]) == 0
