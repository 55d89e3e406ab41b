import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical test")
    # the CPU oracle's fork pool (the reference's ensemble workers) in a
    # process that also runs CUDA threads
    config.addinivalue_line("filterwarnings",
                            "ignore:This process .* is multi-threaded:DeprecationWarning")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    base = os.path.join(REPO, "tests", "golden")
    return {name: np.load(os.path.join(base, name + ".npz"))
            for name in ("kernels", "lorenz", "fhn", "fhnnet", "small")}
