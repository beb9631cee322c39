"""Test configuration: the ``gpu`` marker gates everything that needs a B200.

``python -m pytest tests -m "not gpu"`` runs here (no GPU); ``-m gpu`` runs on
the GPU box through ``gpurun``.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    """Golden vectors written by oracle/gen_golden.py (the reference itself),
    grouped by case: {case: {field: array}}."""
    data = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    cases = {}
    for key in data.files:
        case, field = key.split("/", 1)
        cases.setdefault(case, {})[field] = data[key]
    return cases


@pytest.fixture(scope="session")
def golden():
    return load_golden
