import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libmics.so on cuda:0)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (spawns one process per GPU)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    here = os.path.join(ROOT, "tests", "golden")
    arr = np.load(os.path.join(here, "reference.npz"))
    with open(os.path.join(here, "reference_digests.json")) as fh:
        dig = json.load(fh)
    return arr, dig
