import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libamgb200.so)")
    config.addinivalue_line("markers", "slow: long-running")


def have_reference():
    """The reference package is importable only in the build container."""
    if not os.path.isdir(REF_SRC):
        return False
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    try:
        import amgkit  # noqa: F401
    except Exception:
        return False
    return True


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def _relerr(got, want):
    """Reference acceptance metric (test_acceptance.py:53-57)."""
    import numpy as np

    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(1.0, float(np.abs(want).max(initial=0.0)))
    return float(np.abs(got - want).max(initial=0.0)) / scale
