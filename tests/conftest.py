import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfastwavenet.so")


@pytest.fixture(scope="session")
def built_lib():
    """Builds libfastwavenet.so if stale (nvcc cross-compiles without a GPU)."""
    from paper_1611_09482_b200 import build

    return build.build()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1611_09482_b200 import _lib

    _lib.load()  # fail loudly if the extension is missing
    return torch.device("cuda", 0)
