import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


def _cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _cuda_ok():
        pytest.skip("no CUDA device")
    from paper_2104_06784_b200 import _lib
    return _lib.lib()


@pytest.fixture(scope="session")
def oracle_kind():
    """The CPU checker: the reference itself when oracle/_ref was built, else the C restatement."""
    from oracle import oracle as orc
    if orc.available("ref") or os.path.exists(orc.REF_SOURCES):
        return "ref"
    return "port"
