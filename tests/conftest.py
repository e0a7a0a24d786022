import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# Co-located ranks in one process (test_gpu_multirank) keep several streams
# parked on cuStreamWaitValue32 (push streams, start barrier).  With the
# default 8 hardware work queues, streams share queues and a parked wait can
# block an unrelated stream of another rank; give every stream its own queue.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)
