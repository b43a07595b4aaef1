import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def _gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    """The C restatement (always buildable, travels to the GPU box)."""
    from oracle import Oracle, build

    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build(ref=False)
    return Oracle("c")


@pytest.fixture(scope="session")
def ref_orc():
    """The reference compiled from its own sources (oracle/_ref); skip when absent."""
    from oracle import LIB_REF, Oracle

    if not os.path.exists(LIB_REF):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("ref")
