"""The GPU-metrics sidecar of a reference sweep: the sweep CSV
stays byte-compatible with the reference (its own reader accepts it), the
sidecar is keyed by label. CPU: the reference's row path (FORCE_ROW) where
/root/reference is importable; the B200 tensor path runs in
tests/test_gpu_reference_suite.py."""

import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")


@pytest.fixture
def relab_mod():
    if not REF.exists():
        pytest.skip("reference package not present on this machine")
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    import relab

    yield relab
    sys.path.remove(str(REF))


def test_sweep_csv_stays_reference_compatible_and_sidecar_is_keyed(relab_mod, tmp_path):
    from relab.bench import ExperimentConfig, Operation, read_sweep_csv
    from relab.selector import Policy

    from paper_2602_21237_b200 import sidecar

    g = relab_mod.GenSpec(3000, 500, relab_mod.Uniform(), 8, seed=1)
    cfgs = [ExperimentConfig(Operation.JOIN, g, policy=Policy.FORCE_ROW, repetitions=2, warmup=0, label="j3k",
                             budget=relab_mod.MemoryBudget(1 << 20)),
            ExperimentConfig(Operation.SORT, g, policy=Policy.FORCE_ROW, repetitions=2, warmup=0,
                             budget=relab_mod.MemoryBudget(1 << 20))]
    out = tmp_path / "sweep.csv"
    rows, side = sidecar.sweep_with_sidecar(cfgs, out)
    back = read_sweep_csv(out)  # the reference's reader rejects any extra column
    assert [r.digest_hex for r in back] == [r.digest_hex for r in rows]
    got = sidecar.read_sidecar(str(out) + ".gpu.csv")
    assert [r["label"] for r in got] == ["j3k", sidecar.cell_label(cfgs[1])]
    from oracle import tensorpath_oracle as O

    lk = relab_mod.generate_relation(g).column("key")
    rk = relab_mod.generate_relation(cfgs[0].gen_right).column("key")
    assert got[0]["operation"] == "join" and int(got[0]["output_rows"]) == O.join_count(lk, rk)
    assert float(got[1]["mrows_per_s"]) > 0 and float(got[0]["hbm_frac"]) > 0
    assert int(got[1]["alg_bytes"]) == 3000 * 16 + 3000 * 20
