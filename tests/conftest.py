import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU-oracle runs")
    # Build the checkers (oracle/) and the product library once per session.
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=True, stdout=subprocess.DEVNULL)
    from paper_2109_05072_b200 import build

    build.build()


@pytest.fixture(scope="session")
def golden_equiv():
    idx = json.load(open(os.path.join(GOLDEN, "equivalence.json")))
    arr = np.load(os.path.join(GOLDEN, "equivalence.npz"))
    return idx, arr


@pytest.fixture(scope="session")
def golden_cg():
    return json.load(open(os.path.join(GOLDEN, "cg.json")))
