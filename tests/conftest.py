import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.join(ROOT, "tests")
if TESTS not in sys.path:  # tests/helpers (parity bars, torchrun workers)
    sys.path.insert(0, TESTS)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "ppoff"))


@pytest.fixture(scope="session")
def golden_plans():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "plans.json")) as f:
        return json.load(f)
