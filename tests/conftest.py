import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# Load every kernel module when the CUDA context is created: with lazy loading a
# kernel's first use may synchronize the context, which deadlocks the loopback
# transport's kernel-initiated exchange (a neighbour's put / persistent CG kernel
# spins on this rank while the load waits for it; hofem.h, set_exchange).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built libhofem.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    import json
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def closed(expr: str) -> float:
    """Evaluate a closed-form golden expression like '(1-1/sqrt(5))/2'."""
    import math
    return float(eval(expr, {"__builtins__": {}}, {"sqrt": math.sqrt, "pi": math.pi}))
