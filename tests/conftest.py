import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a device path)")
    config.addinivalue_line("markers", "slow: long CPU parity runs (minutes)")


def _gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    """The reference compiled in place (oracle/_ref); skipped where the
    reference sources and prebuilt shim are both absent (GPU box)."""
    import oracle
    if not oracle.ref_available():
        if not os.path.isdir(oracle.REFERENCE_SRC):
            pytest.skip("reference oracle not built and /root/reference absent")
        oracle.build()
    return oracle.ref_lib()


@pytest.fixture(scope="session")
def hybrid():
    import oracle
    if not oracle.ref_available():
        if not os.path.isdir(oracle.REFERENCE_SRC):
            pytest.skip("reference oracle not built and /root/reference absent")
        oracle.build()
    return oracle.hybrid_lib()


@pytest.fixture(scope="session")
def prod():
    from paper_2410_00428_b200 import _abi
    return _abi.product_lib()


@pytest.fixture(scope="session")
def golden():
    import json
    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "kv_manager.json")) as f:
        kv = json.load(f)
    with open(os.path.join(d, "engine.json")) as f:
        eng = json.load(f)
    return {"kv": kv, "engine": eng}
