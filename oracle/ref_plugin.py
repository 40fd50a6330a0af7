"""pytest plugin — TEST INFRASTRUCTURE ONLY: run the reference's own test
suite (oracle/_ref/relab_tests, built by oracle/build_ref.py) with the B200
operators installed into the live reference package (patch.install(), the
drop-in of SURVEY §8(b) F6). Loaded with ``-p oracle.ref_plugin`` by
tests/test_gpu_reference_suite.py; every tensor-path call the reference's
tests make then runs through librelab_b200.so."""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SITE = ROOT / "oracle" / "_ref" / "site"


def pytest_configure(config):
    for p in (str(SITE), str(ROOT)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import relab  # noqa: F401  (the reference, from oracle/_ref/site)
    import relab.bench  # noqa: F401
    import relab.tensorpath  # noqa: F401

    from paper_2602_21237_b200 import _capi, patch, tensor_path

    _capi.load()  # fail loudly here if the library or the GPU is missing
    replaced = patch.install()
    assert relab.tensor_join is tensor_path.tensor_join and relab.bench.tensor_sort is tensor_path.tensor_sort
    config._rl_replaced = replaced


def pytest_report_header(config):
    n = len(getattr(config, "_rl_replaced", ()))
    return f"relab operators rebound to the B200 drop-in: {n} names (librelab_b200.so)"


def pytest_sessionfinish(session, exitstatus):
    from paper_2602_21237_b200 import _capi

    # evidence that the kernels ran: launches through the library in this process
    sys.stdout.write(f"\n[rl-plugin] librelab_b200 kernel launches: {_capi.load().rl_launch_count()}\n")
