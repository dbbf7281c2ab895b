import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    lib = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    return Oracle(lib)


@pytest.fixture(scope="session")
def reference():
    """The compiled reference (oracle/_ref) or None where it was not built."""
    from oracle.oracle import Reference
    return Reference.load()


@pytest.fixture(scope="session")
def spk():
    import paper_1811_03559_b200 as spk
    from paper_1811_03559_b200 import build
    if not os.path.exists(spk.LIB_PATH):
        build.build()
    spk.lib()
    return spk


def rel_componentwise(a, b):
    """max|a-b| / max(1, max|b|)  (tests/test_util.hpp:100-103)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(1.0, float(np.abs(b).max()))) if a.size else 0.0
