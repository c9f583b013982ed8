"""Test configuration: the ``gpu`` marker and shared helpers.

``-m "not gpu"`` runs on the CPU build container (oracle vs golden vectors,
host logic, C-ABI load/symbol checks, gloo multi-rank host paths);
``-m gpu`` runs on a B200 and calls the CUDA path through the C-ABI.
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
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def relf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb else 1.0))


@pytest.fixture
def golden():
    return load_golden
