import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) configs")


def pytest_collection_modifyitems(config, items):
    # a `-m gpu` run on a box without CUDA must fail loudly, not skip: the GPU
    # tests are the parity gate.  Only the CPU suite may run without a GPU.
    pass


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)
