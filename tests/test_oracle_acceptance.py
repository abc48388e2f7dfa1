"""Pin the CPU oracle to the reference's own acceptance datasets (test_acceptance.py:206-259:
menger-3, the 128^3 shells, 128^3 float blobs x opaque/ramp x 7 index kinds).  CPU only:
classification, every index kind's arrays, and 256x256 frames (pixels + sample counts) of
the oracle equal the unmodified reference's (tests/golden/make_golden.py acceptance)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import (ACCEPT_DATASETS, EQUIV_KINDS, accept_field, oracle_index, render_kind,
                      unpack_bits)
from oracle import oracle as O


class _Cam:
    """Camera.orbit(dims, 30, 15, width=256) without the package (the oracle needs only the
    frame vectors; same float64 expressions as render.py:93-149)."""

    def __init__(self, dims, az=30.0, el=15.0, width=256):
        import math

        center = np.asarray(dims, np.float64) * 0.5
        diameter = float(np.linalg.norm(np.asarray(dims, np.float64)))
        a, e = math.radians(az), math.radians(el)
        u = np.array([math.cos(e) * math.sin(a), math.sin(e), math.cos(e) * math.cos(a)])
        self.eye = center + diameter * u
        d = center - self.eye
        self.direction = d / float(np.linalg.norm(d))
        r = np.cross(self.direction, np.array([0.0, 1.0, 0.0]))
        r = r / float(np.linalg.norm(r))
        up = np.cross(r, self.direction)
        self.up = up / float(np.linalg.norm(up))
        self.extent = diameter
        self.width = self.height = width


@pytest.mark.parametrize("dname", ACCEPT_DATASETS)
@pytest.mark.parametrize("tname", ["opaque", "ramp"])
def test_oracle_acceptance_structures_and_frames(acceptance, dname, tname):
    g = acceptance
    field, dims = accept_field(g, dname)
    key = f"{dname}_{tname}"
    lut = g[f"{tname}_lut"]
    bits, plain = O.classify(field, lut, dilate=True)
    assert plain == int(g[f"{key}_plain_count"])
    np.testing.assert_array_equal(bits, unpack_bits(g[f"{key}_bits"], dims))
    cam = _Cam(dims)
    rgba, samples = O.render("naive", field, lut, None, cam)
    np.testing.assert_array_equal(O.quantize_rgba(rgba), g[f"{key}_naive_pixels"])
    assert int(samples.sum()) == int(g[f"{key}_naive_samples"])
    for kind in EQUIV_KINDS:
        k = f"{key}_{kind}"
        idx = oracle_index(O, kind, bits)
        if kind == "grid":
            np.testing.assert_array_equal(idx["occupied"], g[f"{k}_occupied"])
        else:
            tree = idx["tree"] if kind == "hybrid" else idx
            for f in ("lo", "hi", "left", "right") + (
                    ("leaf_brick", "brick_coords") if kind == "lbvh" else ("axis", "plane")):
                np.testing.assert_array_equal(tree[f], g[f"{k}_{f}"], err_msg=f"{k}.{f}")
            assert tree["height"] == int(g[f"{k}_height"])
        if kind == "hybrid":
            np.testing.assert_array_equal(idx["occupied"], g[f"{k}_occupied"])
        rgba, samples = O.render(render_kind(kind), field, lut, idx, cam)
        np.testing.assert_array_equal(O.quantize_rgba(rgba), g[f"{k}_pixels"], err_msg=k)
        assert int(samples.sum()) == int(g[f"{k}_samples"]), k


def test_oracle_thin_shell_sampling_reduction(acceptance):
    """Criterion 7 (test_acceptance.py:237-259): kd-deep-mls32 takes <= 20% of naive's samples
    on the thin shell; the oracle's counts equal the reference's."""
    g = acceptance
    field, dims = accept_field(g, "thinshell128")
    lut = g["opaque_lut"]
    bits, _ = O.classify(field, lut, dilate=True)
    np.testing.assert_array_equal(bits, unpack_bits(g["thinshell128_opaque_bits"], dims))
    cam = _Cam(dims)
    _, naive = O.render("naive", field, lut, None, cam)
    _, kd = O.render("kd", field, lut, oracle_index(O, "kd-deep-mls32", bits), cam)
    assert int(naive.sum()) == int(g["thinshell128_opaque_naive_samples"])
    assert int(kd.sum()) == int(g["thinshell128_opaque_kd-deep-mls32_samples"])
    assert kd.sum() / naive.sum() <= 0.20
