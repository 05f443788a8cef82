import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs under `-m gpu`")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    r = Reference()
    if not r.available:
        pytest.skip("oracle/_ref/libsfref.so not built (reference tree absent)")
    return r


@pytest.fixture(scope="session")
def sf():
    """The product package; on a GPU box the CUDA library MUST load (no fallback)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_06095_b200.sparsefuse as sfm
    sfm.lib()  # raises if the library is missing
    return sfm
