import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built libmns_b200.so")


class Golden:
    """Reference-generated fixtures (oracle/gen_golden.py) stored as npz + a JSON manifest."""

    def __init__(self, name):
        self.z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
        self.manifest = json.loads(str(self.z["manifest"]))

    def __getitem__(self, key):
        return self.z[key]


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]

    return get


def cfg_tuple(cfg):
    inf = float("inf")
    e = tuple(inf if cfg[k] is None else cfg[k] for k in ("e1", "e2", "e3"))
    return e, cfg["mean_tol"], cfg["mode"] == "mns"
