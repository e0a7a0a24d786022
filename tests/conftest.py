import os
import subprocess
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
    config.addinivalue_line("markers", "isolated(timeout): run the test in its own process, killed after timeout s")


@pytest.hookimpl(tryfirst=True)
def pytest_pyfunc_call(pyfuncitem):
    """Tests marked `isolated` run in a child pytest process with a hard
    timeout: a hang there (e.g. co-located ranks) fails that test
    instead of stalling the whole suite."""
    mark = pyfuncitem.get_closest_marker("isolated")
    if mark is None or os.environ.get("MXP_ISOLATED_CHILD"):
        return None
    timeout = mark.kwargs.get("timeout", 300)
    env = dict(os.environ, MXP_ISOLATED_CHILD="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu or not gpu",
           pyfuncitem.nodeid]
    try:
        r = subprocess.run(cmd, cwd=ROOT, env=env, timeout=timeout, capture_output=True, text=True)
    except subprocess.TimeoutExpired:
        pytest.fail(f"isolated test process killed after {timeout} s (hang)")
    if r.returncode != 0:
        pytest.fail("isolated test failed:\n" + r.stdout[-4000:] + r.stderr[-2000:])
    return True


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)
