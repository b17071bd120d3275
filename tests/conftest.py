import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    """The C port is tiny; (re)build it if missing. The reference wrapper is
    built only where /root/reference exists (never on the GPU box, which gets
    the prebuilt oracle/_ref/*.so through gpurun)."""
    from oracle import oracle as O
    if not O.available("port") or (os.path.isdir(O.REF_SRC) and not O.available("ref")):
        O.build()
    yield


def require_ref():
    from oracle import oracle as O
    if not O.available("ref"):
        pytest.skip("oracle/_ref/libep_ref.so not built (reference tree absent)")


@pytest.fixture(scope="session")
def cuda_handle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_11729_b200 import Handle
    return Handle(0)
