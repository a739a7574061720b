import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as _oracle
    _oracle.lib()
    return _oracle


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def mandel():
    """The product binding; on a GPU box a missing extension is a hard error."""
    from paper_2007_00745_b200 import mandel as _m
    _m.lib()
    return _m


@pytest.fixture(scope="session")
def cuda_ok():
    if not _cuda_available():
        pytest.fail("a -m gpu test ran without a CUDA device")
    return True
