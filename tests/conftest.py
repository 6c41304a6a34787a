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
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden_small():
    """{case_name: {key: array}} from tests/golden/golden_small.npz (reference-generated)."""
    z = np.load(os.path.join(GOLDEN, "golden_small.npz"))
    cases = {}
    for k in z.files:
        name, key = k.split("__", 1)
        cases.setdefault(name, {})[key] = z[k]
    return cases


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"golden_{name}.npz"))
    return {k: z[k] for k in z.files}


def golden_b(case):
    if "B" in case:
        return case["B"]
    if "B_seed" in case:
        return np.random.default_rng(int(case["B_seed"])).random(tuple(case["B_shape"]))
    return None


MEDIUM = ["cfg1_full", "cfg2b_s16", "cfg4_s8", "cfg5_s32", "rmat12_t3", "rmat12_t9", "rmat16_t7"]


@pytest.fixture(scope="session")
def golden_small():
    return load_golden_small()


@pytest.fixture
def rng():
    return np.random.default_rng(20240917)
