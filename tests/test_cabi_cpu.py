"""CPU checks of the C ABI: libvsb200.so loads without a GPU, exports every function that
include/vsb200.h declares, and its host-only helpers (TF parameter block, Morton side) behave."""

from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vsb200.h"
LIB = ROOT / "paper_1912_09596_b200" / "libvsb200.so"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_1912_09596_b200 import _build

        _build.build()
    return C.CDLL(str(LIB))


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(vs_[a-z0-9_]+)$", out, flags=re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(lib, n)


def test_python_binding_covers_header():
    from paper_1912_09596_b200._lib import SIGNATURES

    missing = [n for n in declared() if n not in SIGNATURES]
    assert not missing, missing


def _params(lib, alpha):
    buf = np.zeros(16, np.int32)
    a = np.ascontiguousarray(alpha, np.float32)
    assert lib.vs_tf_params_from_alpha(C.c_void_p(a.ctypes.data), C.c_void_p(buf.ctypes.data)) == 0
    return buf


@pytest.mark.parametrize("kind", ["ramp", "band", "low", "comb", "all", "none", "twoband"])
def test_tf_params(lib, kind):
    a = np.zeros(256, np.float32)
    if kind == "ramp":
        a[154:] = 0.5
    elif kind == "band":
        a[100:151] = 0.3
    elif kind == "low":
        a[:99] = 1.0
    elif kind == "comb":
        a[::17] = 1.0
    elif kind == "all":
        a[:] = 0.1
    elif kind == "twoband":
        a[10:13] = 0.5
        a[250:] = 0.25
    p = _params(lib, a)
    vis = a > 0
    words = [int(sum(int(vis[32 * w + k]) << k for k in range(32))) for w in range(8)]
    assert [int(x) & 0xFFFFFFFF for x in p[:8]] == words
    flips = [b for b in range(1, 256) if vis[b] != vis[b - 1]]
    mode, start = int(p[8]), int(p[9])
    assert start == int(vis[0])
    assert int(p[12]) == int(vis.sum())
    if not flips:
        assert mode == 3
    elif len(flips) <= 2:
        assert mode == len(flips) and list(p[10:10 + len(flips)]) == flips
    else:
        assert mode == 0


def test_morton_side(lib):
    assert lib.vs_morton_side(1, 1, 1) == 8
    assert lib.vs_morton_side(128, 128, 128) == 128
    assert lib.vs_morton_side(64, 63, 64) == 64
    assert lib.vs_morton_side(65, 2, 3) == 128
    assert lib.vs_morton_side(1025, 1, 1) < 0


def test_version(lib):
    lib.vs_version.restype = C.c_char_p
    assert b"sm_100a" in lib.vs_version()


def _last_error(lib) -> str:
    buf = C.create_string_buffer(512)
    lib.vs_last_error(buf, C.c_size_t(512))
    return buf.value.decode()


def test_argument_errors_without_gpu(lib):
    """The status convention (include/vsb200.h): argument errors return a negative status and
    name the entry point in vs_last_error, before any device work (so they run on CPU)."""
    dummy = C.c_void_p(0x1000)  # never dereferenced: validation fails first
    i = C.c_int
    cases = [
        ("vs_classify_bits", lambda: lib.vs_classify_bits(None, i(8), i(8), i(8), None, None, None, None)),
        ("vs_classify_dilate_bits", lambda: lib.vs_classify_dilate_bits(
            dummy, i(8), i(8), i(33), dummy, dummy, None, None)),
        ("vs_dilate_bits", lambda: lib.vs_dilate_bits(dummy, i(4), i(4), i(4), dummy, None)),
        ("vs_kd_build", lambda: lib.vs_kd_build(None, i(8), i(8), i(8), i(0), i(-1), i(0), i(4),
                                                i(8), None, None)),
        ("vs_build_mquads", lambda: lib.vs_build_mquads(dummy, i(5), i(8), i(8), i(8), dummy, None)),
        ("vs_render", lambda: lib.vs_render(None, None, None, None, None, C.c_double(0.5), i(0),
                                            None, None, None, None, None, None, None,
                                            C.c_size_t(0), i(0), None, None)),
    ]
    for name, fn in cases:
        st = fn()
        assert st < 0, (name, st)
        assert name in _last_error(lib), (name, _last_error(lib))
