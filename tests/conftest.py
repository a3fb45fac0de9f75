import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path through the C-ABI")


@pytest.fixture(scope="session")
def restatement():
    from oracle import Restatement

    return Restatement()


@pytest.fixture(scope="session")
def reference():
    """The compiled, unmodified reference (oracle/_ref); skipped where it was not built."""
    from oracle import REFERENCE_SO, Reference

    if not os.path.exists(REFERENCE_SO):
        pytest.skip("oracle/_ref/libbnmc_ref.so not built")
    return Reference()


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, name + ".npz"))
