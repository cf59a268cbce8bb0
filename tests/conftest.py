import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


@pytest.fixture(scope="session")
def orc():
    """The C restatement of the reference (oracle/fmafft_oracle.c)."""
    import oracle
    return oracle.load_oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference library itself (oracle/_ref), when it was built here."""
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.load_ref()


@pytest.fixture(scope="session")
def dsfft():
    import paper_2604_00567_b200 as d
    d._load()
    return d


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
