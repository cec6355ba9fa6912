import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The in-process multi-rank tests run up to four fake ranks on ONE device,
# each with a main and a side stream whose copy-engine halo uses stream
# memory-op waits (peer_halo.cu).  With the default 8 hardware work queues
# the ~10 streams alias onto shared queues, and a blocked wait at the head of
# a queue can hold back the very work it waits for (an intermittent hang of
# the P = 4 copy-engine cases).  One process per GPU (the product) uses 2-3
# streams and never aliases; the tests get a queue per stream.  Must be set
# before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (large sizes)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "paper_spec_examples.json")) as f:
        return json.load(f)
