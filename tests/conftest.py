import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libdcx.so)")
    config.addinivalue_line("markers", "slow: long-running")


@lru_cache(maxsize=1)
def golden():
    with open(GOLDEN / "golden.json") as f:
        return json.load(f)


@lru_cache(maxsize=1)
def golden_arrays():
    return dict(np.load(GOLDEN / "golden_arrays.npz"))


@pytest.fixture(scope="session")
def gold():
    return golden()


@pytest.fixture(scope="session")
def garr():
    return golden_arrays()


@lru_cache(maxsize=1)
def golden_k2():
    """K2000 over all 1024 seeds (tests/golden/make_golden_k2.py): per-seed best energy,
    iterations, stop reason (0 converged, 1 max_iters, 2 time_budget) and the best-so-far
    improvement points, DOCH and ADOCH."""
    with open(GOLDEN / "golden_k2.json") as f:
        g = json.load(f)
    g["arrays"] = dict(np.load(GOLDEN / "golden_k2.npz"))
    return g


@pytest.fixture(scope="session")
def gk2():
    return golden_k2()


@pytest.fixture(scope="session")
def pgold():
    """Procedural-coupling fixtures (tests/golden/make_golden_procedural.py)."""
    with open(GOLDEN / "golden_procedural.json") as f:
        g = json.load(f)
    g["arrays"] = dict(np.load(GOLDEN / "golden_procedural.npz"))
    return g


@lru_cache(maxsize=None)
def g1_csr():
    from paper_2509_01928_b200 import synth

    return synth.g1_shape()


@lru_cache(maxsize=None)
def k2_W():
    from paper_2509_01928_b200 import synth

    return synth.dense_pm1(2000, seed=20240817)


@lru_cache(maxsize=None)
def sk_dense(n, seed):
    from paper_2509_01928_b200 import synth

    return synth.sk_gaussian(n, seed)
