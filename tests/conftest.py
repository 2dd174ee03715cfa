import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA extension")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    g = os.path.join(ROOT, "tests", "golden")
    return {n: dict(np.load(os.path.join(g, n + ".npz"))) for n in ("kat", "ops", "attention", "lengths", "next")}
