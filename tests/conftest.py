import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    torch.cuda.init()
    return torch.device("cuda:0")


class _Knobs:
    """Library experiment knobs (ngemm_cuda_set_option): the library reads NGEMM_* from the
    environment once, so tests switch kernels through the C-ABI and reset after each test."""

    def set(self, name, value):
        from paper_1910_00178_b200 import _lib
        if name == "I16_PATH":
            value = {"tcgen05": 1, "simt": 0}.get(value, value)
        _lib.set_option(name, int(value))


@pytest.fixture
def knobs():
    yield _Knobs()
    from paper_1910_00178_b200 import _lib
    _lib.reset_options()
