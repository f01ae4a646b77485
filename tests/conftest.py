import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden_sweeps():
    with open(os.path.join(GOLDEN, "sweeps.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN, "sweeps.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def golden_runs():
    with open(os.path.join(GOLDEN, "runs.json")) as fh:
        return {r["name"]: r for r in json.load(fh)}


@pytest.fixture(scope="session")
def golden_solvers():
    return np.load(os.path.join(GOLDEN, "solvers.npz"))


@pytest.fixture
def rng():
    return np.random.default_rng(20240911)
