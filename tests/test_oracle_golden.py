"""Pin the CPU oracle (oracle/vs_oracle.c) to golden vectors from the unmodified reference.

CPU only.  These are the tests that make the oracle trustworthy: every structure and render
the GPU path is later compared against is first shown here to equal the reference's output
bit for bit (structures, pixels, sample counts) and exactly (float RGBA).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import unpack_bits
from oracle import oracle as O

TREE_F = ("lo", "hi", "left", "right")


def _check_tree(got: dict, gold: dict, prefix: str):
    for f in TREE_F:
        np.testing.assert_array_equal(got[f], gold[f"{prefix}_{f}"], err_msg=f"{prefix}.{f}")
    if f"{prefix}_axis" in gold:
        np.testing.assert_array_equal(got["axis"], gold[f"{prefix}_axis"])
        np.testing.assert_array_equal(got["plane"], gold[f"{prefix}_plane"])
    else:
        np.testing.assert_array_equal(got["leaf_brick"], gold[f"{prefix}_leaf_brick"])
        np.testing.assert_array_equal(got["brick_coords"], gold[f"{prefix}_brick_coords"])
    assert got["root"] == int(gold[f"{prefix}_root"])
    assert got["height"] == int(gold[f"{prefix}_height"])


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


def check_structures(gold: dict, prefix: str):
    dims = tuple(int(d) for d in gold[prefix + "dims"])
    bits = unpack_bits(gold[prefix + "bits"], dims)
    coords, codes = O.flag_bricks(bits, 8)
    np.testing.assert_array_equal(coords, gold[prefix + "brick_coords_scan"])
    np.testing.assert_array_equal(codes, gold[prefix + "brick_codes_scan"])
    _check_tree(O.build_lbvh(coords, codes, 8, dims), gold, prefix + "lbvh")
    np.testing.assert_array_equal(O.macro_grid(bits, 16), gold[prefix + "grid16"])
    for key in gold:
        if key.startswith(prefix + "svt") and key[len(prefix) + 3:].isdigit():
            bs = int(key[len(prefix) + 3:])
            np.testing.assert_array_equal(O.svt_build(bits, bs), gold[key], err_msg=key)
    cells = O.cell_boxes(bits, 8)
    for f in ("codes", "coords", "lo", "hi", "occupied"):
        np.testing.assert_array_equal(cells[f], gold[prefix + f"cells8_{f}"], err_msg=f)
    for name, kw in KD_ARGS.items():
        if prefix + name + "_lo" in gold:
            _check_tree(O.kd_build(bits, **kw), gold, prefix + name)
    return bits


@pytest.mark.parametrize("tname", ["ramp03", "ramp06", "ramp00", "opaque", "band"])
def test_blobs64_classify_and_structures(blobs64, tname):
    u8 = blobs64["u8"]
    lut = blobs64[f"{tname}_lut"]
    plain, cnt = O.classify(u8, lut, dilate=False)
    np.testing.assert_array_equal(plain, unpack_bits(blobs64[f"{tname}_plain_bits"], u8.shape))
    assert cnt == int(blobs64[f"{tname}_plain_count"])
    assert cnt / u8.size == float(blobs64[f"{tname}_occupancy"])
    dil, _ = O.classify(u8, lut, dilate=True)
    np.testing.assert_array_equal(dil, unpack_bits(blobs64[f"{tname}_bits"], u8.shape))
    check_structures(blobs64, f"{tname}_")


@pytest.mark.parametrize("case", ["rand_64x48x40", "rand_20x17x9", "blocky48", "blocky_37x45x50", "sparse64"])
def test_bit_cases_structures(bitcases, case):
    check_structures(bitcases, f"{case}_")


@pytest.mark.parametrize("scene", ["shell", "menger"])
@pytest.mark.parametrize("tname", ["opaque", "ramp"])
def test_scene_structures(scenes, scene, tname):
    check_structures(scenes, f"{scene}_{tname}_")


class _Cam:
    def __init__(self, g, w, h):
        self.eye = tuple(g["cam_eye"]); self.direction = tuple(g["cam_dir"]); self.up = tuple(g["cam_up"])
        self.extent = float(g["cam_extent"]); self.width = w; self.height = h


def _index(kind, gold, prefix, dims):
    if kind == "naive":
        return "naive", None
    if kind == "grid":
        return "grid", {"occupied": gold[prefix + "grid16"], "cell_size": 16}
    def tree(p):
        t = {f: gold[f"{p}_{f}"] for f in TREE_F}
        for f in ("axis", "plane", "leaf_brick"):
            if f"{p}_{f}" in gold:
                t[f] = gold[f"{p}_{f}"]
        t["root"] = int(gold[f"{p}_root"]); t["height"] = int(gold[f"{p}_height"])
        return t
    if kind == "lbvh":
        return "lbvh", tree(prefix + "lbvh")
    if kind == "hybrid":
        return "hybrid", {"occupied": gold[prefix + "grid16"], "cell_size": 16, "tree": tree(prefix + "kd-shallow")}
    return "kd", tree(prefix + kind)


def test_camera_origins_match(blobs64):
    cam = _Cam(blobs64, 96, 64)
    packed, d = O.camera_vectors(cam)
    eye, up, right, scale = packed[:3], packed[3:6], packed[6:9], packed[9]
    xs = (np.arange(96) + 0.5 - 96 / 2.0) * scale
    ys = (64 / 2.0 - np.arange(64) - 0.5) * scale
    o = (eye[None, None, :] + ys[:, None, None] * up[None, None, :]) + xs[None, :, None] * right[None, None, :]
    np.testing.assert_array_equal(o.reshape(-1, 3), blobs64["cam_origins"])


@pytest.mark.parametrize("tname", ["ramp03", "band"])
@pytest.mark.parametrize("kind", ["naive", "grid", "lbvh", "kd-shallow", "kd-deep-mls32", "kd-binned-mls32", "hybrid"])
def test_blobs64_render_exact(blobs64, tname, kind):
    """Float RGBA and per-pixel sample counts equal the reference's bit for bit."""
    cam = _Cam(blobs64, 96, 64)
    k, idx = _index(kind, blobs64, f"{tname}_", (64, 64, 64))
    rgba, samples = O.render(k, blobs64["u8"], blobs64[f"{tname}_lut"], idx, cam, nthreads=4)
    np.testing.assert_array_equal(samples, blobs64[f"{tname}_render_{kind}_samples"])
    np.testing.assert_array_equal(rgba, blobs64[f"{tname}_render_{kind}_rgba"])
    np.testing.assert_array_equal(O.quantize_rgba(rgba), blobs64[f"{tname}_render_{kind}_pixels"])


class _OrbitCam:
    """Camera.orbit (render.py:93-132) restated for the scene fixtures."""

    def __init__(self, dims, az, el, width, height=None):
        center = np.asarray(dims, dtype=np.float64) * 0.5
        diameter = float(np.linalg.norm(np.asarray(dims, dtype=np.float64)))
        a, e = math.radians(az), math.radians(max(-89.9, min(89.9, el)))
        u = np.array([math.cos(e) * math.sin(a), math.sin(e), math.cos(e) * math.cos(a)])
        eye = center + diameter * u
        d = (center - eye) / float(np.linalg.norm(center - eye))
        right = np.cross(d, np.array([0.0, 1.0, 0.0]))
        right = right / float(np.linalg.norm(right))
        up = np.cross(right, d)
        up = up / float(np.linalg.norm(up))
        self.eye, self.direction, self.up = tuple(eye), tuple(d), tuple(up)
        self.extent, self.width, self.height = diameter, width, height or width


@pytest.mark.parametrize("scene", ["shell", "menger"])
@pytest.mark.parametrize("tname", ["opaque", "ramp"])
def test_scene_frames_exact(scenes, scene, tname):
    u8 = scenes[f"{scene}_u8"]
    cam = _OrbitCam(u8.shape, 25.0, 20.0, 64)
    lut = scenes[f"{scene}_{tname}_lut"]
    for kind in ("naive", "grid", "lbvh", "kd-deep-mls32", "hybrid"):
        k, idx = _index(kind, scenes, f"{scene}_{tname}_", u8.shape)
        rgba, samples = O.render(k, u8, lut, idx, cam, nthreads=4)
        np.testing.assert_array_equal(O.quantize_rgba(rgba), scenes[f"{scene}_{tname}_render_{kind}_pixels"])
        assert int(samples.sum()) == int(scenes[f"{scene}_{tname}_render_{kind}_samples"])
    if tname == "ramp":
        rgba, samples = O.render("naive", u8, lut, None, cam, nearest=True, nthreads=4)
        np.testing.assert_array_equal(O.quantize_rgba(rgba), scenes[f"{scene}_ramp_render_nearest_pixels"])
        assert int(samples.sum()) == int(scenes[f"{scene}_ramp_render_nearest_samples"])


def test_float_volume_render_exact(misc):
    data = misc["f32_data"]
    lut = misc["f32_lut"]
    dil, _ = O.classify(data, lut, dilate=True)
    np.testing.assert_array_equal(dil, unpack_bits(misc["f32_dil_bits"], data.shape))
    assert O.classify(data, lut)[1] == int(misc["f32_plain_count"])
    cam = _OrbitCam(data.shape, 40.0, -20.0, 32, 24)
    coords, codes = O.flag_bricks(dil, 8)
    for kind, idx in (("naive", None), ("lbvh", O.build_lbvh(coords, codes, 8, data.shape)),
                      ("kd", O.kd_build(dil, mode="deep"))):
        rgba, samples = O.render(kind, data, lut, idx, cam, nthreads=2)
        np.testing.assert_array_equal(samples, misc[f"f32_render_{kind}_samples"])
        np.testing.assert_array_equal(rgba, misc[f"f32_render_{kind}_rgba"])


def test_single_ray_traversal_and_integrate(blobs64):
    dims = (64, 64, 64)
    for kind, key in (("naive", None), ("grid", "grid"), ("lbvh", "lbvh"), ("kd", "kd-deep-mls32"), ("hybrid", "hybrid")):
        k, idx = _index(key or "naive", blobs64, "ramp03_", dims)
        counts = blobs64[f"trav_{kind}_counts"]
        segs = blobs64[f"trav_{kind}_segs"]
        off = 0
        for o, d, c in zip(blobs64["rays_o"], blobs64["rays_d"], counts):
            got = O.traverse(k, idx, dims, o, d)
            np.testing.assert_array_equal(got, segs[off:off + c], err_msg=kind)
            off += c
    off = 0
    for r, (o, d) in enumerate(zip(blobs64["rays_o"], blobs64["rays_d"])):
        segs = O.traverse("naive", None, dims, o, d)
        rgba, n = O.integrate(o, d, segs, blobs64["u8"], blobs64["ramp03_lut"])
        np.testing.assert_array_equal(rgba, blobs64["integrate_rgba"][r])
        assert n == int(blobs64["integrate_samples"][r])


def test_snapped_positions_and_morton(misc):
    for row in misc["snapped"]:
        lo, hi, bins, cs, n = (int(v) for v in row[:5])
        assert O.snapped_positions(lo, hi, bins, cs) == [int(v) for v in row[5:5 + n]]
    assert O.morton_encode(0, 0, 0) == 0 and O.morton_encode(1, 1, 1) == 7 and O.morton_encode(3, 0, 0) == 9


def test_corr_table_is_libm_pow(misc, blobs64):
    lut = blobs64["ramp03_lut"]
    np.testing.assert_array_equal(O.corr_table(lut, 0.5)[lut[:, 3] > 0], misc["corr_ramp03_dt05"][lut[:, 3] > 0])
    np.testing.assert_array_equal(O.corr_table(lut, 0.5), O.math_pow_corr(lut, 0.5))


def test_u8_quantisation_is_identity():
    assert O.quantize_u8_identity()


def test_shrink_direct_equals_svt(rng):
    """or_tight_box (direct scan, used inside the k-d oracle) == shrink_to_occupied via SVT."""
    bits = rng.random((40, 33, 29)) < 0.01
    for bs in (8, 32):
        t = O.svt_build(bits, bs)
        for _ in range(60):
            lo = rng.integers(0, 30, size=3)
            hi = lo + rng.integers(1, 20, size=3)
            assert O.shrink_svt(t, bits.shape, bs, lo, hi) == O.tight_box(bits, lo, hi)
            want = int(bits[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].sum())
            assert O.box_count(t, bits.shape, bs, lo, hi) == want


@pytest.mark.parametrize("kind", ["naive", "lbvh"])
def test_multichannel_oracle_reduces_to_reference(blobs64, kind):
    """With channels 1..3 at zero alpha the multi-channel restatement IS the reference frame
    (the only pinned case of the multi-channel semantics, which the reference lacks)."""
    cam = _Cam(blobs64, 96, 64)
    u8 = blobs64["u8"]
    zero = np.zeros((256, 4), np.float32)
    k, idx = _index(kind, blobs64, "ramp03_", (64, 64, 64))
    rgba, samples = O.render_multi(k, [u8, u8[::-1].copy(), u8, u8.T.copy()],
                                   [blobs64["ramp03_lut"], zero, zero, zero], idx, cam)
    np.testing.assert_array_equal(samples, blobs64[f"ramp03_render_{kind}_samples"])
    np.testing.assert_array_equal(rgba, blobs64[f"ramp03_render_{kind}_rgba"])
