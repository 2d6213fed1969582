import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfeastb200.so")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE config)")


@pytest.fixture(scope="session")
def unit_golden():
    return np.load(os.path.join(GOLDEN, "unit.npz"))


@pytest.fixture(scope="session")
def small_golden():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_symmetric(n, rng, scale=1.0):
    r = rng.normal(size=(n, n))
    return scale * (r + r.T) / 2.0


def random_hermitian(n, rng, scale=1.0):
    r = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    return scale * (r + r.conj().T) / 2.0


def gap_interval(evals, lo, hi):
    evals = np.sort(evals)
    emin = evals[lo] - 1.0 if lo == 0 else 0.5 * (evals[lo - 1] + evals[lo])
    emax = evals[hi] + 1.0 if hi == len(evals) - 1 else 0.5 * (evals[hi] + evals[hi + 1])
    return float(emin), float(emax)
