import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"

try:
    from hypothesis import settings
    settings.register_profile("suite", deadline=None, max_examples=25)
    settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: large configs")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    meta = json.loads((GOLDEN / "reference_meta.json").read_text())
    arrays = np.load(GOLDEN / "reference_cases.npz")
    return meta, arrays


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)
