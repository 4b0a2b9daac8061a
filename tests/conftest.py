import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_SRC = os.path.join(ROOT, "baseline", "_ref", "src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def ref():
    """The reference package (this container only; never on the GPU box)."""
    if not os.path.isdir(os.path.join(REF_SRC, "tweedmg")):
        pytest.skip("reference tweedmg not built in baseline/_ref")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import tweedmg
    return tweedmg


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
