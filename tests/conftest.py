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


def pytest_collection_modifyitems(config, items):
    """A plain `pytest` on a machine without a GPU skips the gpu-marked tests.

    An explicit `-m gpu` run never skips: there the module fixtures assert a
    CUDA device, so a GPU box that lost its device fails loudly instead of
    passing on nothing.
    """
    if "gpu" in (config.getoption("-m") or "").replace("not gpu", ""):
        return
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="needs a CUDA device (run with -m gpu on a B200)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


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
