import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long CPU oracle runs; set HJ_SLOW=1 to run")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("HJ_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow oracle run; set HJ_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)
