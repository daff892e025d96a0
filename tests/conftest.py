import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-cube / large-size checks")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_outputs.npz"))


@pytest.fixture(scope="session")
def figures():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "figures.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def caching_golden():
    """lut caching variant + approximant evaluators from the live reference (make_golden.py --caching-only)."""
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "caching_outputs.npz"))
