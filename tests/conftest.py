"""Shared test setup.

* registers the `gpu` marker (tests needing a B200; run with -m gpu);
* pins OPENBLAS to one thread so oracle norms match the golden fixtures,
  which were produced by the real reference with OPENBLAS_NUM_THREADS=1
  (SURVEY.md F2);
* puts the repo root on sys.path so `oracle` and the package import.
"""

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import json  # noqa: E402
import sys  # noqa: E402

import numpy as np  # noqa: E402
import pytest  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

# numpy may already be imported by a pytest plugin before this file runs, so
# the environment variable alone is not enough: limit the live BLAS pools.
_BLAS_LIMIT = threadpool_limits(limits=1, user_api="blas")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_exists(name):
    return os.path.exists(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def golden_stencils():
    return load_json("stencils.json")
