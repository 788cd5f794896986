import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


def reference_available() -> bool:
    """The unmodified reference package built by oracle/build_ref.sh."""
    return os.path.isdir(os.path.join(REPO, "oracle", "_ref", "gemmforge"))


def import_reference():
    path = os.path.join(REPO, "oracle", "_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    import gemmforge  # noqa: F401

    return gemmforge


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(REPO, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def small_cases():
    import numpy as np

    return dict(np.load(os.path.join(REPO, "tests", "golden", "small_cases.npz")))
