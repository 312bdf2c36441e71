import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
_GOLDEN = os.path.join(ROOT, "tests", "golden")  # bigtrack.fits
if _GOLDEN not in sys.path:
    sys.path.append(_GOLDEN)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "reference: needs the Python reference under /root/reference")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "ixverify"))


@pytest.fixture(scope="session")
def reference():
    """The reference package (only present in the build container)."""
    if not have_reference():
        pytest.skip("reference (/root/reference) not present on this machine")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import ixverify.oracle as oracle  # noqa: F401

    return sys.modules["ixverify"]


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_23058_b200 import _lib

    _lib.load(require_device=True)  # fails loudly if libixgpu.so is missing
    return torch.device("cuda:0")
