"""Shared test configuration.  `gpu` tests need a B200 (run on the GPU box via
gpurun); everything else runs on CPU here."""
import os
import sys

import pytest

# Emulated ranks put one proxy agent stream (plus an op stream) per rank on
# one device; with more streams than hardware queues an agent stream can alias
# onto the queue of the MoE kernel it must feed (csrc/proxy.cu).  Before any
# CUDA context exists:
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

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
