"""Shared test configuration.  `gpu` tests need a B200 (run on the GPU box via
gpurun); everything else runs on CPU here."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def gpu_count():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0
