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


# PCG history tolerance, entry by entry: |h_k - ref_k| <= REL * ref_k +
# FLOOR * ref_0.  The dot products are reordered sums (a fixed-order device
# tree vs OpenBLAS ddot), so alpha and beta differ in the last bits and CG,
# which does not damp such perturbations, carries absolute differences of a
# few hundred ulp of the INITIAL scale into every later iterate (the
# attainable accuracy of finite-precision CG is O(eps ||A|| ||x||)).  Entry
# k therefore agrees to ~eps * ref_0 / ref_k relative: 1e-6 relative while
# the measure is above ~1e-7 of its start, and FLOOR * ref_0 = 1e-13 of the
# start (~450 ulp; 0.1 % of the last entry of a 1e10 solve) beyond.  The
# FMA build also rounds every preconditioner application differently, and
# its n = 12 tails reach 1.5e-13 of the start: its floor is 1e-12.
PCG_REL, PCG_FLOOR, PCG_FLOOR_FAST = 1e-6, 1e-13, 1e-12


def check_pcg_hist(hist, ref_h, floor=PCG_FLOOR):
    hist, ref_h = np.asarray(hist), np.asarray(ref_h[: len(hist)])
    assert len(hist) == len(ref_h)
    d = np.abs(hist - ref_h)
    assert np.max(d) / ref_h[0] < 1e-10
    bound = PCG_REL * np.abs(ref_h) + floor * ref_h[0]
    assert np.all(d <= bound), (float(np.max(d / bound)), int(np.argmax(d / bound)), len(hist))
    return float(np.max(d / np.abs(ref_h)))
