import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def solver():
    from paper_2412_08346_b200 import Solver

    s = Solver()
    yield s
    s.close()


@pytest.fixture(scope="session")
def oracle():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return ref
