"""The reference's OWN tests and harness on the B200 through the drop-in
(VERDICT r1 "missing" 3).

oracle/_ref (built by oracle/build_ref.py from /root/reference/pkg, shipped
with the working tree) holds the unmodified `relab` package and its test
directory. Here
* its whole pytest suite runs with the B200 operators installed
  (oracle/ref_plugin.py -> patch.install()): test_tensorpath.py,
  test_selector.py, test_oracles.py, test_bench.py and the rest;
* its harness `run_experiment` runs cfg1 on the tensor path with 50 and 100
  repetitions — every repetition's multiset digest must agree
  (bench.py:254-260, DigestMismatch) — and the report equals the one the
  reference's CPU tensor path produces (same digest, rows, path choice,
  peak_mem_bytes).
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import build_ref  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not build_ref.available(), reason="oracle/_ref not built (no /root/reference here)")]


def test_reference_test_suite_passes_on_the_b200_operators():
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "oracle.ref_plugin", "-p", "no:cacheprovider",
                        "-x", str(build_ref.TESTS)], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    passed = int(re.search(r"(\d+) passed", out).group(1))
    assert passed >= 120, out[-2000:]
    launches = int(re.search(r"\[rl-plugin\] librelab_b200 kernel launches: (\d+)", out).group(1))
    assert launches > 1000  # the tensor-path tests really ran on the kernels


@pytest.fixture(scope="module")
def relab_patched():
    sys.path.insert(0, str(build_ref.SITE))
    import relab
    import relab.bench

    from paper_2602_21237_b200 import patch

    yield relab
    patch.uninstall()


@pytest.mark.parametrize("reps", [50, 100])
def test_run_experiment_cfg1_digest_stable(relab_patched, reps):
    relab = relab_patched
    from relab.bench import ExperimentConfig, Operation, run_experiment
    from relab.selector import Policy

    from paper_2602_21237_b200 import patch

    gen = relab.GenSpec(1_000_000, 1_000_000, relab.Uniform(), 8, seed=0)
    cfg = ExperimentConfig(Operation.JOIN, gen, policy=Policy.FORCE_TENSOR, repetitions=reps, warmup=3,
                           label="cfg1-b200")
    patch.uninstall()
    ref = run_experiment(ExperimentConfig(Operation.JOIN, gen, policy=Policy.FORCE_TENSOR, repetitions=1, warmup=0))
    patch.install()
    rep = run_experiment(cfg)  # DigestMismatch if any repetition differs
    assert rep.output_rows == ref.output_rows == 1_000_488
    assert rep.result_digest == ref.result_digest
    assert rep.path_taken == ref.path_taken
    assert rep.spill == ref.spill  # zero spill, the reference's peak_mem_bytes formula
    assert len(rep.latency.samples) == reps


def test_run_experiment_sort_matches_reference(relab_patched):
    relab = relab_patched
    from relab.bench import ExperimentConfig, Operation, run_experiment
    from relab.selector import Policy

    from paper_2602_21237_b200 import patch

    gen = relab.GenSpec(2_000_000, 2**62, relab.Uniform(), 4, seed=3)
    mk = lambda r: ExperimentConfig(Operation.SORT, gen, policy=Policy.FORCE_TENSOR, repetitions=r, warmup=0)  # noqa
    patch.uninstall()
    ref = run_experiment(mk(1))
    patch.install()
    rep = run_experiment(mk(5))
    assert rep.result_digest == ref.result_digest and rep.output_rows == ref.output_rows
    assert rep.spill == ref.spill


def test_reference_sweep_with_gpu_sidecar(relab_patched, tmp_path):
    """relab's sweep on the B200 tensor path, its CSV unchanged (the
    reference's reader), the GPU metrics in the sidecar keyed by label."""
    relab = relab_patched
    from relab.bench import ExperimentConfig, Operation, read_sweep_csv
    from relab.selector import Policy

    from paper_2602_21237_b200 import patch, sidecar

    patch.install()
    g = relab.GenSpec(500_000, 500_000, relab.Uniform(), 8, seed=2)
    cfgs = [ExperimentConfig(Operation.JOIN, g, policy=Policy.FORCE_TENSOR, repetitions=5, warmup=1, label="j"),
            ExperimentConfig(Operation.SORT, g, policy=Policy.FORCE_TENSOR, repetitions=5, warmup=1, label="s")]
    rows, side = sidecar.sweep_with_sidecar(cfgs, tmp_path / "sw.csv")
    assert [r.path_taken for r in read_sweep_csv(tmp_path / "sw.csv")] == ["tensor", "tensor"]
    got = sidecar.read_sidecar(str(tmp_path / "sw.csv") + ".gpu.csv")
    assert [r["label"] for r in got] == ["j", "s"] and all(r["gpus"] == "1" for r in got)
    assert all(float(r["mrows_per_s"]) > 0 for r in got)
