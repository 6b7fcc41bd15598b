import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built extension")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        info = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, name + ".npz"))
    return info, arrays


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)
