import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libzk.so")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_cases(data):
    """Group 'case__field' keys into {case: {field: array}}."""
    out = {}
    for key, val in data.items():
        case, field = key.split("__", 1)
        out.setdefault(case, {})[field] = val
    return out


@pytest.fixture(scope="session")
def vecops_golden():
    return golden_cases(load_golden("vecops"))


@pytest.fixture(scope="session")
def spmv_golden():
    return golden_cases(load_golden("spmv"))


@pytest.fixture(scope="session")
def bicgstab_golden():
    return golden_cases(load_golden("bicgstab"))


@pytest.fixture(scope="session")
def problems_golden():
    return golden_cases(load_golden("problems"))
