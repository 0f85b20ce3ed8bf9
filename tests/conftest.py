"""Shared fixtures.  `-m gpu` tests need a B200 and call the C-ABI engine;
everything else runs on CPU (oracle vs golden vectors, host logic, ABI load)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def scenario(name):
    from paper_2210_07297_b200 import problem as P
    if name == "synthetic96":
        return P.synthetic_c4()
    return P.load_scenario(os.path.join(GOLDEN, "scenarios", name + ".json"))


def hexf(s):
    return float.fromhex(s)


@pytest.fixture(scope="session")
def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
