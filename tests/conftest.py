import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    import numpy as np
    return np.load(os.path.join(GOLDEN, name))


def group(npz, prefix):
    """{key: array} for the keys 'prefix/<key>' of a golden archive."""
    return {k[len(prefix) + 1:]: npz[k] for k in npz.files if k.startswith(prefix + "/")}


def cases(npz):
    return sorted({k.split("/")[0] for k in npz.files})


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O
