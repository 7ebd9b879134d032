"""Shared test setup.  `-m "not gpu"` runs here (no GPU): oracle vs reference/goldens, host policy
logic through the C ABI, ABI symbol checks.  `-m gpu` runs on a B200: the CUDA path vs the goldens
and the oracle."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def load_golden(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        return json.load(f)


def golden_names():
    return sorted(n[:-5] for n in os.listdir(GOLDEN) if n.endswith(".json") and n != "MANIFEST.json")


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False
