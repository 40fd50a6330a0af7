import os
import sys
from pathlib import Path

import pytest
from hypothesis import HealthCheck, settings

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

# the reference's hypothesis profile (pkg/tests/conftest.py:1-9)
settings.register_profile("relab", deadline=None, max_examples=60, suppress_health_check=[HealthCheck.too_slow])
settings.load_profile("relab")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through librelab_b200.so)")
    config.addinivalue_line("markers", "slow: large CPU-side oracle work (seconds)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    meta = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    arrays = dict(np.load(ROOT / "tests" / "golden" / "golden.npz"))
    return meta["cases"], arrays
