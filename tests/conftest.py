"""Test configuration: registers the ``gpu`` marker and makes sure the in-tree
CUDA library is built before the package is imported (nvcc cross-compiles
sm_100a without a GPU; ``make`` is a no-op when the .so is up to date)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

LIB = os.path.join(ROOT, "paper_2107_02671_b200", "lib", "libsincfft_b200.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")
    if not os.path.exists(LIB) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(ROOT, "paper_2107_02671_b200", "csrc")], check=True)


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")

    def load(name):
        return np.load(os.path.join(d, name), allow_pickle=False)
    return load
