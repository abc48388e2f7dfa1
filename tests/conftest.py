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


@pytest.fixture(scope="session")
def acceptance():
    """The reference's acceptance datasets (test_acceptance.py:206-259) through the unmodified
    reference: inputs, every index kind's arrays, 256x256 frames (make_golden.acceptance)."""
    return _load("acceptance.npz")


ACCEPT_DATASETS = ("menger3", "shell128", "blobs128")
EQUIV_KINDS = ("grid", "lbvh", "kd-shallow", "kd-deep-mls32", "kd-deep-mls128",
               "kd-binned-mls32", "hybrid")
KD_ARGS = {
    "kd-shallow": dict(mode="shallow"),
    "kd-deep": dict(mode="deep"),
    "kd-deep-mls8": dict(mode="deep", max_leaf_size=8),
    "kd-deep-mls32": dict(mode="deep", max_leaf_size=32),
    "kd-deep-mls128": dict(mode="deep", max_leaf_size=128),
    "kd-binned-mls32": dict(mode="deep", max_leaf_size=32, builder="binned"),
    "kd-binned": dict(mode="deep", builder="binned"),
    "kd-binned-mls8": dict(mode="deep", max_leaf_size=8, builder="binned"),
}


def accept_field(gold, dname):
    """(array the oracle takes, dims): u8 bins for u8-exact datasets, else the float field."""
    a = gold[f"{dname}_u8"] if f"{dname}_u8" in gold else gold[f"{dname}_f32"]
    return a, a.shape


def oracle_index(O, kind, bits):
    """The oracle's index of ``kind`` as the dict O.render takes."""
    if kind == "naive":
        return None
    if kind == "grid":
        return {"occupied": O.macro_grid(bits, 16), "cell_size": 16}
    if kind == "lbvh":
        coords, codes = O.flag_bricks(bits, 8)
        return O.build_lbvh(coords, codes, 8, bits.shape)
    if kind == "hybrid":
        return {"occupied": O.macro_grid(bits, 16), "cell_size": 16,
                "tree": O.kd_build(bits, **KD_ARGS["kd-shallow"])}
    return O.kd_build(bits, **KD_ARGS[kind])


def render_kind(kind):
    return "kd" if kind.startswith("kd-") else kind
