import os
import sys

# Sharded groups put several ranks on the one test GPU (tests/test_gpu_shard.py):
# each rank's streams need their own hardware queue (skg_shard_group_init checks).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU-only test")


@pytest.fixture(scope="session")
def orc64():
    from oracle.oracle import Oracle
    return Oracle("f64")


@pytest.fixture(scope="session")
def orc32():
    from oracle.oracle import Oracle
    return Oracle("f32")
