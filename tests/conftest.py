import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU sweeps (exhaustive 2^32); opt-in with -m slow")


def pytest_collection_modifyitems(config, items):
    # slow tests run only when selected explicitly (-m slow or -m "slow and ...")
    expr = config.getoption("-m") or ""
    if "slow" in expr:
        return
    skip = pytest.mark.skip(reason="slow: select with -m slow")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
