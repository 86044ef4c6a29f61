import os
import sys

import pytest

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # see paper_2510_19470_b200/__init__.py

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    # Make sure the in-tree libraries exist (incremental make; seconds when up to date).
    import __graft_entry__ as g

    g.build(import_package=False)


def _cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def record_accuracy(request):
    """record_accuracy(**errors): appends the observed errors of a parity test to the JSON
    lines file named by HEP_ACCURACY_LOG (if set) -- the data the stated tolerances
    (tests/tolerances.py) are set from."""
    import json

    def rec(**vals):
        path = os.environ.get("HEP_ACCURACY_LOG")
        if path:
            with open(path, "a") as f:
                f.write(json.dumps({"test": request.node.nodeid, **vals}) + "\n")

    return rec
