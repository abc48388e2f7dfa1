"""GPU parity of classification, brick flags, LBVH and macro grid (csrc/classify.cu, lbvh.cu).

Every device result is compared bit for bit with the golden vectors produced by the
unmodified reference (tests/golden) and, for random inputs, with the CPU oracle
(oracle/vs_oracle.c) that test_oracle_golden.py pins to those vectors.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import unpack_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    return vs


def _check_lbvh(idx, gold, prefix):
    for f in ("lo", "hi", "left", "right", "leaf_brick", "brick_coords"):
        np.testing.assert_array_equal(getattr(idx, f), gold[f"{prefix}_{f}"], err_msg=f)
    assert idx.root == int(gold[f"{prefix}_root"])
    assert idx.height() == int(gold[f"{prefix}_height"])


def _check_lbvh_oracle(idx, ref):
    for f in ("lo", "hi", "left", "right", "leaf_brick", "brick_coords"):
        np.testing.assert_array_equal(getattr(idx, f), ref[f], err_msg=f)
    assert idx.root == ref["root"]
    assert idx.height() == ref["height"]


@pytest.mark.parametrize("tname", ["ramp03", "ramp06", "ramp00", "opaque", "band"])
def test_blobs64_classify_bricks_lbvh_grid(vs, blobs64, tname):
    u8 = blobs64["u8"]
    tf = vs.TransferFunction(blobs64[f"{tname}_lut"])
    v = vs.Volume.from_u8(u8)
    plain = vs.classify(v, tf, dilate=False)
    np.testing.assert_array_equal(plain.bits, unpack_bits(blobs64[f"{tname}_plain_bits"], u8.shape))
    assert vs.occupancy(vs.classify(v, tf)) == float(blobs64[f"{tname}_occupancy"])
    dil = vs.classify(v, tf, dilate=True)
    # fused summary path (lazy classification, 8^3 bricks)
    bricks = vs.flag_bricks(dil, 8)
    np.testing.assert_array_equal(bricks.coords, blobs64[f"{tname}_brick_coords_scan"])
    np.testing.assert_array_equal(bricks.codes, blobs64[f"{tname}_brick_codes_scan"])
    _check_lbvh(vs.build_lbvh(bricks), blobs64, f"{tname}_lbvh")
    np.testing.assert_array_equal(vs.derive_macro_grid(dil, 16).occupied, blobs64[f"{tname}_grid16"])
    # materialised bits path
    np.testing.assert_array_equal(dil.bits, unpack_bits(blobs64[f"{tname}_bits"], u8.shape))
    b = vs.BinaryVolume(dil.bits)
    bricks2 = vs.flag_bricks(b, 8)
    np.testing.assert_array_equal(bricks2.coords, blobs64[f"{tname}_brick_coords_scan"])
    _check_lbvh(vs.build_lbvh(bricks2), blobs64, f"{tname}_lbvh")
    np.testing.assert_array_equal(vs.derive_macro_grid(b, 16).occupied, blobs64[f"{tname}_grid16"])


@pytest.mark.parametrize("case", ["rand_64x48x40", "rand_20x17x9", "blocky48", "blocky_37x45x50", "sparse64"])
def test_bit_cases(vs, bitcases, case):
    p = f"{case}_"
    dims = tuple(int(d) for d in bitcases[p + "dims"])
    bits = unpack_bits(bitcases[p + "bits"], dims)
    b = vs.BinaryVolume(bits)
    np.testing.assert_array_equal(b.bits, bits)
    bricks = vs.flag_bricks(b, 8)
    np.testing.assert_array_equal(bricks.coords, bitcases[p + "brick_coords_scan"])
    np.testing.assert_array_equal(bricks.codes, bitcases[p + "brick_codes_scan"])
    _check_lbvh(vs.build_lbvh(bricks), bitcases, p + "lbvh")
    # generic BrickSet path (host-built, CUB sort)
    hand = vs.BrickSet(8, dims, bitcases[p + "brick_coords_scan"], bitcases[p + "brick_codes_scan"])
    _check_lbvh(vs.build_lbvh(hand), bitcases, p + "lbvh")
    np.testing.assert_array_equal(vs.derive_macro_grid(b, 16).occupied, bitcases[p + "grid16"])


@pytest.mark.parametrize("scene", ["shell", "menger"])
@pytest.mark.parametrize("tname", ["opaque", "ramp"])
def test_scenes(vs, scenes, scene, tname):
    p = f"{scene}_{tname}_"
    u8 = scenes[f"{scene}_u8"]
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction(scenes[p + "lut"])
    dil = vs.classify(v, tf, dilate=True)
    dims = u8.shape
    np.testing.assert_array_equal(dil.bits, unpack_bits(scenes[p + "bits"], dims))
    bricks = vs.flag_bricks(vs.classify(v, tf, dilate=True), 8)
    np.testing.assert_array_equal(bricks.coords, scenes[p + "brick_coords_scan"])
    _check_lbvh(vs.build_lbvh(bricks), scenes, p + "lbvh")
    np.testing.assert_array_equal(vs.derive_macro_grid(dil, 16).occupied, scenes[p + "grid16"])


def _band_lut(lo, hi):
    lut = np.zeros((256, 4), np.float32)
    lut[:, 0] = np.linspace(0, 1, 256)
    lut[lo:hi + 1, 3] = 0.5
    return lut


@pytest.mark.parametrize("dims", [(48, 40, 64), (64, 64, 32), (33, 17, 48), (24, 24, 528),
                                  (40, 70, 96), (7, 33, 1024)])
@pytest.mark.parametrize("tfkind", ["ramp", "ramp_lo", "band", "band_mid", "band_lo", "low", "lowhi",
                                    "twoband", "comb", "all", "none"])
def test_random_volumes_vs_oracle(vs, rng, dims, tfkind):
    """Fused summary path (all four visibility modes) vs the oracle on blocky random u8."""
    nx, ny, nz = dims
    coarse = rng.integers(0, 256, size=(-(-nx // 5), -(-ny // 5), -(-nz // 5)), dtype=np.uint8)
    u8 = np.repeat(np.repeat(np.repeat(coarse, 5, 0), 5, 1), 5, 2)[:nx, :ny, :nz].copy()
    noise = rng.integers(0, 256, size=dims, dtype=np.uint8)
    mask = rng.random(dims) < 0.01
    u8[mask] = noise[mask]
    if tfkind == "ramp":
        lut = vs.TransferFunction.ramp(0.8).lut
    elif tfkind == "ramp_lo":
        lut = vs.TransferFunction.ramp(0.2).lut
    elif tfkind == "band":
        lut = _band_lut(200, 203)
    elif tfkind == "band_mid":
        lut = _band_lut(100, 150)
    elif tfkind == "band_lo":
        lut = _band_lut(10, 12)
    elif tfkind == "low":
        lut = _band_lut(0, 99)
    elif tfkind == "lowhi":
        lut = _band_lut(0, 199)
    elif tfkind == "twoband":
        lut = _band_lut(10, 12)
        lut[250:, 3] = 0.25
    elif tfkind == "comb":
        lut = np.zeros((256, 4), np.float32)
        lut[::17, 3] = 1.0
    elif tfkind == "all":
        lut = np.full((256, 4), 0.5, np.float32)
    else:
        lut = np.zeros((256, 4), np.float32)
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction(lut)
    ref_plain, cnt = O.classify(u8, lut, dilate=False)
    ref_dil, _ = O.classify(u8, lut, dilate=True)
    for dilate, ref in ((False, ref_plain), (True, ref_dil)):
        b = vs.classify(v, tf, dilate=dilate)
        bricks = vs.flag_bricks(b, 8)
        coords, codes = O.flag_bricks(ref, 8)
        np.testing.assert_array_equal(bricks.coords, coords)
        np.testing.assert_array_equal(bricks.codes, codes)
        _check_lbvh_oracle(vs.build_lbvh(bricks), O.build_lbvh(coords, codes, 8, dims))
        np.testing.assert_array_equal(vs.derive_macro_grid(vs.classify(v, tf, dilate=dilate), 16).occupied,
                                      O.macro_grid(ref, 16))
        np.testing.assert_array_equal(b.bits, ref)
    assert vs.classify(v, tf).base_count() == cnt
    # warm path: from its second dilated TF on, a volume votes from its per-brick halo presence
    # masks (vs_presence_to_bitmap) instead of reading the voxels -- same bricks, tree, grid
    assert "_presence" in v.__dict__
    bw = vs.classify(v, tf, dilate=True)
    bricks = vs.flag_bricks(bw, 8)
    coords, codes = O.flag_bricks(ref_dil, 8)
    np.testing.assert_array_equal(bricks.coords, coords)
    np.testing.assert_array_equal(bricks.codes, codes)
    idx = vs.build_lbvh(bricks)
    _check_lbvh_oracle(idx, O.build_lbvh(coords, codes, 8, dims))
    nb = [-(-d // 8) for d in dims]
    grid_bits = np.unpackbits(idx.brick_grid().cpu().numpy().view(np.uint8), bitorder="little")
    want = np.zeros(nb[0] * nb[1] * nb[2], np.uint8)
    want[(coords[:, 0] * nb[1] + coords[:, 1]) * nb[2] + coords[:, 2]] = 1
    np.testing.assert_array_equal(grid_bits[:want.size], want)
    assert not grid_bits[want.size:].any()
    # packed dilated bits first (the fused classify+dilate pass when nz % 32 == 0): same bits,
    # and the undilated count comes out of the same pass
    b = vs.classify(v, tf, dilate=True)
    b.packed()
    np.testing.assert_array_equal(b.bits, ref_dil)
    assert b.base_count() == cnt


@pytest.mark.parametrize("bs", [1, 3, 8, 16])
def test_brick_sizes_vs_oracle(vs, rng, bs):
    dims = (37, 45, 50)
    bits = rng.random(dims) < 0.002
    b = vs.BinaryVolume(bits)
    bricks = vs.flag_bricks(b, bs)
    coords, codes = O.flag_bricks(bits, bs)
    np.testing.assert_array_equal(bricks.coords, coords)
    np.testing.assert_array_equal(bricks.codes, codes)
    _check_lbvh_oracle(vs.build_lbvh(bricks), O.build_lbvh(coords, codes, bs, dims))
    for cs in (2, 5, 16):
        np.testing.assert_array_equal(vs.derive_macro_grid(b, cs).occupied, O.macro_grid(bits, cs))


def test_edge_cases(vs):
    dims = (16, 16, 16)
    empty = vs.BinaryVolume(np.zeros(dims, bool))
    bricks = vs.flag_bricks(empty)
    assert bricks.count == 0 and bricks.coords.shape == (0, 3)
    idx = vs.build_lbvh(bricks)
    assert idx.node_count == 0 and idx.root == -1 and idx.height() == 0
    one = np.zeros((32, 32, 32), bool)
    one[17, 9, 25] = True  # test_lbvh.py:132-139
    idx = vs.build_lbvh(vs.flag_bricks(vs.BinaryVolume(one)))
    assert idx.node_count == 1 and idx.root == 0 and idx.height() == 1
    np.testing.assert_array_equal(idx.lo[0], [16, 8, 24])
    np.testing.assert_array_equal(idx.hi[0], [24, 16, 32])
    # codes 0..3 -> 7 nodes, height 3 (test_lbvh.py:142-151)
    coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.int32)
    codes = vs.morton_encode(coords[:, 0], coords[:, 1], coords[:, 2])
    idx = vs.build_lbvh(vs.BrickSet(8, (16, 16, 8), coords, codes))
    assert idx.node_count == 7 and idx.height() == 3
    # duplicate codes: ties broken by the scan index
    dup = vs.BrickSet(8, (64, 64, 64), np.array([[1, 1, 1]] * 3 + [[0, 0, 0]], np.int32),
                      np.array([7, 7, 7, 0], np.uint32))
    ref = O.build_lbvh(dup.coords, dup.codes, 8, (64, 64, 64))
    _check_lbvh_oracle(vs.build_lbvh(dup), ref)


def test_float_volume_quantisation(vs, misc):
    data = misc["f32_data"]
    lut = misc["f32_lut"]
    v = vs.Volume(data)
    assert v.field is not None  # not u8-representable: the renderer keeps the float field
    b = vs.classify(v, vs.TransferFunction(lut), dilate=True)
    np.testing.assert_array_equal(b.bits, unpack_bits(misc["f32_dil_bits"], data.shape))
    assert vs.classify(v, vs.TransferFunction(lut)).base_count() == int(misc["f32_plain_count"])
    edge = np.array([0.0, 1.0, 0.5, -0.25, 1.5, np.nan, 0.5 / 255, 1.5 / 255], np.float32)
    vv = vs.Volume(np.tile(edge, (2, 2, 1)))
    np.testing.assert_array_equal(vv.bins.cpu().numpy()[0, 0], vs.quantize_scalar(edge))


@pytest.mark.parametrize("dims", [(40, 36, 128), (17, 33, 256), (32, 16, 1024)])
def test_macro_grid_from_bits_vs_oracle(vs, rng, dims):
    """16^3 cell votes over packed bits (whole-word rows: the vectorised vote kernel) and the
    k-d root box from the same bits, against the oracle."""
    bits = rng.random(dims) < 0.0007
    b = vs.BinaryVolume(bits)
    np.testing.assert_array_equal(vs.derive_macro_grid(b, 16).occupied, O.macro_grid(bits, 16))
    kd = vs.build_kdtree(vs.build_svt_grid(b), vs.BuildParams(mode="shallow"))
    ref = O.kd_build(bits, mode="shallow")
    for f in ("lo", "hi", "axis", "plane", "left", "right"):
        np.testing.assert_array_equal(getattr(kd, f), ref[f])


@pytest.mark.parametrize("dims,world", [((64, 48, 32), 2), ((72, 40, 48), 3), ((40, 24, 16), 8)])
def test_presence_slab_shards_equal_full_build(vs, dims, world):
    """vs_presence_build_slab over each rank's brick x-slabs (tiles.presence_slabs, uneven and
    empty ranges included) writes exactly the words of the full build; with no process group
    tiles.shard_presence is the plain Volume.presence()."""
    import torch

    from paper_1912_09596_b200 import _lib
    from paper_1912_09596_b200.tiles import presence_slabs, shard_presence

    rng = np.random.default_rng(sum(dims) + world)
    u8 = rng.integers(0, 256, dims, dtype=np.uint8)
    u8[rng.random(dims) < 0.7] = 0
    v = vs.Volume.from_u8(u8)
    full = v.presence().clone()
    nx, ny, nz = dims
    nbx = -(-nx // 8)
    parts = torch.full_like(full, -7)
    for bx0, bx1 in presence_slabs(nbx, world):
        _lib.call("vs_presence_build_slab", _lib.ptr(v.bins), nx, ny, nz, bx0, bx1,
                  _lib.ptr(parts), _lib.stream())
    torch.cuda.synchronize()
    assert torch.equal(parts, full)
    with pytest.raises(_lib.VsError):
        _lib.call("vs_presence_build_slab", _lib.ptr(v.bins), nx, ny, nz, 0, nbx + 1,
                  _lib.ptr(parts), _lib.stream())
    assert torch.equal(shard_presence(v), full)
