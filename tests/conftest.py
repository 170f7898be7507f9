import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (seconds to minutes)")


@pytest.fixture(scope="session")
def coracle():
    from oracle import c_oracle
    return c_oracle.load()


@pytest.fixture(scope="session")
def phe():
    """The product binding (CUDA path).  GPU tests only: it fails loudly without the .so."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_07329_b200 as phe_mod
    phe_mod.load()  # raises if libphe.so is missing: no silent fallback
    return phe_mod
