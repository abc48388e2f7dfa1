"""Shared fixtures.  ``-m gpu`` tests need a CUDA device and the built libvsb200.so; everything
else runs on CPU (oracle vs golden vectors, host logic, C-ABI symbol checks, gloo ws=2)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def _load(name):
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def blobs64():
    return _load("blobs64.npz")


@pytest.fixture(scope="session")
def scenes():
    return _load("scenes.npz")


@pytest.fixture(scope="session")
def bitcases():
    return _load("bits.npz")


@pytest.fixture(scope="session")
def misc():
    return _load("misc.npz")


def unpack_bits(packed, dims):
    n = int(np.prod(dims))
    return np.unpackbits(packed)[:n].reshape(tuple(int(d) for d in dims)).astype(bool)


@pytest.fixture()
def rng():
    return np.random.default_rng(12345)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
