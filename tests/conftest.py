import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _load(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


@pytest.fixture(scope="session")
def golden_kat():
    return _load("kat.npz")


@pytest.fixture(scope="session")
def golden_grid_fft():
    return _load("grid_fft.npz")


@pytest.fixture(scope="session")
def golden_grid_naive():
    return _load("grid_naive.npz")


@pytest.fixture(scope="session")
def golden_configs():
    return _load("configs.npz")


@pytest.fixture(scope="session")
def golden_counts():
    with open(os.path.join(GOLDEN, "counts.json")) as fh:
        return json.load(fh)["rows"]
