import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libpasd_b200.so")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.lib()  # builds liboracle.so on first use
    return oracle


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    import paper_1712_09999_b200 as pb

    pb.lib()
    return pb
