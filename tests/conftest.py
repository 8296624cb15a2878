"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a
B200 through gpurun.  GPU tests never skip silently: without a CUDA device
they fail (the product path has no CPU fallback)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size checks")


@pytest.fixture(scope="session")
def golden():
    with np.load(os.path.join(GOLDEN, "golden.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def hashes():
    with open(os.path.join(GOLDEN, "hashes.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle import orc as o

    o.build()
    return o


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device: the B200 path has no CPU fallback")
    from paper_1002_4482_b200 import _native

    _native.lib()
    return torch.device("cuda", 0)


@pytest.fixture
def sg_env(monkeypatch):
    """Set SG_* experiment switches for one test: the library parses them
    once, so every change is followed by sg_tuning_reload(), and the
    defaults are restored (and reloaded) when the test ends."""
    from paper_1002_4482_b200 import _native

    def set_(**kv):
        for k, v in kv.items():
            monkeypatch.setenv(k, str(v))
        _native.lib().sg_tuning_reload()

    yield set_
    monkeypatch.undo()
    _native.lib().sg_tuning_reload()
