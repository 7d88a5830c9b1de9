import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libstg.so")


@pytest.fixture(scope="session")
def ctx():
    import paper_2603_29235_b200 as stg
    c = stg.Context(0)
    yield c
    c.close()
