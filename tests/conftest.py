import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_allocator():
    with open(os.path.join(GOLDEN, "allocator_scripts.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_store():
    with open(os.path.join(GOLDEN, "store_scripts.json")) as f:
        metas = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN, "store_scripts.npz")))
    return metas, arrays


@pytest.fixture(scope="session")
def golden_attention():
    with open(os.path.join(GOLDEN, "attention_cases.json")) as f:
        index = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN, "attention_cases.npz")))
    return index, arrays


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "pagedkv"))


@pytest.fixture(scope="session")
def live_reference():
    """The real reference package, importable only in the build container."""
    if not reference_available():
        pytest.skip("reference tree not mounted (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import pagedkv

    return pagedkv
