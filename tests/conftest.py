import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle
    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle
    if not pyoracle.Ref.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return pyoracle.Ref()


@pytest.fixture(scope="session")
def checker():
    """Best available CPU checker: the compiled reference, else the C restatement."""
    from oracle import pyoracle
    return pyoracle.best_checker()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_12485_b200 as hfz
    c = hfz.Context(0)
    yield c
    c.close()
