import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdrcb.so")


def load_golden(name):
    d = dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))
    for k in list(d):
        if k == "cfg" or k.startswith("doc"):
            d[k] = json.loads(bytes(d[k]).decode("utf-8"))
    return d


@pytest.fixture(scope="session")
def golden():
    return load_golden
