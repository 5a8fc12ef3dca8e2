import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) -- the parity tests proper")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) parity runs")
    import buildlib

    buildlib.build_synth()
    buildlib.build_oracle()


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def cuda_device():
    if not has_cuda():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback exists)")
    import torch

    return torch.device("cuda:0")
