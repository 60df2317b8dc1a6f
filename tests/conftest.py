import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as O

    if not O.have_port():
        pytest.skip("oracle/liboracle.so not built (run __graft_entry__.build())")
    return O


def pytest_sessionfinish(session, exitstatus):
    """PARITY_REPORT=<path>: write every parity check's record (tests/parity.py)."""
    path = os.environ.get("PARITY_REPORT")
    if not path:
        return
    try:
        import json

        import parity

        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(parity.RECORDS, f, indent=1)
    except Exception as e:  # never fail the session over the report
        print("parity report not written:", e)
