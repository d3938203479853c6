import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def hx(s):
    return float.fromhex(s)


def untag(t):
    return t[1] if t[0] == "i" else float.fromhex(t[1])


@pytest.fixture(scope="session")
def router_cases():
    return golden("router_cases.json")


@pytest.fixture(scope="session")
def router_replays():
    return golden("router_replays.json")


@pytest.fixture(scope="session")
def phase1_cases():
    return golden("phase1_cases.json")


@pytest.fixture(scope="session")
def cuda_ready():
    try:
        import torch
    except ImportError:
        pytest.skip("torch missing")
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return True
