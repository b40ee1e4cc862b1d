import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the dsdv C-ABI)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref_oracle():
    from oracle.oracle_lib import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


@pytest.fixture(scope="session")
def verifier():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_11733_b200.dsdv import Verifier
    return Verifier(0)
