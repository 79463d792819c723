"""Test configuration.

Markers: ``gpu`` — needs a CUDA device (run on the B200 with ``-m gpu``); everything else
runs on CPU (``-m "not gpu"``).  The TEST-ONLY checkers under oracle/ (the reference compiled
out-of-tree, oracle/_ref/libtsref.so, and the C restatement oracle/liboracle.so) are loaded
here as checkers only.
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def _load(name):
    with open(os.path.join(GOLDEN_DIR, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    return _load("golden.json")


@pytest.fixture(scope="session")
def golden_big():
    p = os.path.join(GOLDEN_DIR, "golden_big.json")
    if not os.path.exists(p):
        pytest.skip("golden_big.json not generated")
    return _load("golden_big.json")


@pytest.fixture(scope="session")
def small_cases():
    return dict(np.load(os.path.join(GOLDEN_DIR, "small_cases.npz")))


@pytest.fixture(scope="session")
def port():
    from oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("reference build oracle/_ref/libtsref.so absent (needs /root/reference)")
    return Ref()


@pytest.fixture(scope="session")
def ts():
    import paper_1502_00355_b200 as mod
    return mod


@pytest.fixture(scope="session")
def capi():
    from paper_1502_00355_b200 import capi as c
    return c


@pytest.fixture(scope="session")
def gpu_ctx(capi):
    if capi.lib().tsg_device_count() <= 0:
        pytest.fail("gpu test selected but no CUDA device is visible")
    return capi.Context(0)
