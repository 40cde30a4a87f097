import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the loopback tests run up to 2 kernels per logical rank concurrently (its stream and its
# exchange stream) whose CTAs meet at peer flags: with the default 8 hardware work queues
# two of those streams can share a queue, serialising a waiting kernel in front of the one
# it waits for.  32 queues (the maximum) give every stream its own (set before CUDA init).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
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
