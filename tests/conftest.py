import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def reference_rsr():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference checkout not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import rsr  # noqa: F401
    return rsr
