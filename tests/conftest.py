"""Shared fixtures.  Markers: ``gpu`` (needs a B200; run with -m gpu) and
``slow`` (multi-minute CPU oracle runs)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running oracle comparisons")


def golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".npz"):
        return np.load(path, allow_pickle=False)
    import json

    with open(path) as fh:
        return json.load(fh)


@pytest.fixture
def rng():
    return np.random.default_rng(20240611)


@pytest.fixture(scope="session")
def oracle_lib():
    """Build oracle/liboracle.so once (CPU checker)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import port

    return port


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():  # -m gpu must not pass silently
        pytest.fail("no CUDA device: the B200 path has no CPU fallback")
    import paper_2006_13053_b200 as pkg

    pkg._native.lib()
    return pkg
