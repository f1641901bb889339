import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")   # pip install of the reference (git-ignored)
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.append(REF)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs the CUDA path through the C ABI")
    config.addinivalue_line("markers", "slow: longer GPU parity cases")


def have_streamcut() -> bool:
    try:
        import streamcut  # noqa: F401
        return True
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
