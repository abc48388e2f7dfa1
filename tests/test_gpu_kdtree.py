"""GPU parity of the summed-volume tables, box queries, k-d trees (sweep and binned) and the
hybrid index (csrc/svt.cu, csrc/kdtree.cu) against the reference's golden vectors and the
CPU oracle: every array bit for bit, rows in the reference's DFS preorder."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import unpack_bits
from oracle import oracle as O

pytestmark = pytest.mark.gpu

KD_PARAMS = {
    "kd-shallow": dict(mode="shallow"),
    "kd-deep": dict(mode="deep"),
    "kd-deep-mls8": dict(mode="deep", max_leaf_size=8),
    "kd-deep-mls32": dict(mode="deep", max_leaf_size=32),
    "kd-deep-mls128": dict(mode="deep", max_leaf_size=128),
    "kd-binned-mls32": dict(mode="deep", max_leaf_size=32, builder="binned"),
    "kd-binned": dict(mode="deep", builder="binned"),
    "kd-binned-mls8": dict(mode="deep", max_leaf_size=8, builder="binned"),
}


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    return vs


def _check_tree(t, want: dict, msg=""):
    for f in ("lo", "hi", "axis", "plane", "left", "right"):
        np.testing.assert_array_equal(getattr(t, f), want[f], err_msg=f"{msg}.{f}")
    assert t.root == want["root"], msg
    assert t.height() == want["height"], msg


def _gold_tree(g, p):
    return {f: g[f"{p}_{f}"] for f in ("lo", "hi", "axis", "plane", "left", "right")} | {
        "root": int(g[f"{p}_root"]), "height": int(g[f"{p}_height"])}


def _structures(vs, g, prefix, b):
    g_svt = None
    for key in g:
        if key.startswith(prefix + "svt") and key[len(prefix) + 3:].isdigit():
            bs = int(key[len(prefix) + 3:])
            svt = vs.build_svt_grid(b, bs)
            np.testing.assert_array_equal(svt.tables, g[key], err_msg=key)
            if bs == 32:
                g_svt = svt
    svt = g_svt or vs.build_svt_grid(b, 32)
    for name, kw in KD_PARAMS.items():
        if prefix + name + "_lo" in g:
            t = vs.build_kdtree(svt, vs.BuildParams(**kw))
            _check_tree(t, _gold_tree(g, prefix + name), prefix + name)


@pytest.mark.parametrize("tname", ["ramp03", "ramp06", "ramp00", "opaque", "band"])
def test_blobs64(vs, blobs64, tname):
    v = vs.Volume.from_u8(blobs64["u8"])
    b = vs.classify(v, vs.TransferFunction(blobs64[f"{tname}_lut"]), dilate=True)
    _structures(vs, blobs64, f"{tname}_", b)


@pytest.mark.parametrize("case", ["rand_64x48x40", "rand_20x17x9", "blocky48", "blocky_37x45x50",
                                  "sparse64"])
def test_bit_cases(vs, bitcases, case):
    dims = tuple(int(d) for d in bitcases[f"{case}_dims"])
    b = vs.BinaryVolume(unpack_bits(bitcases[f"{case}_bits"], dims))
    _structures(vs, bitcases, f"{case}_", b)


@pytest.mark.parametrize("scene", ["shell", "menger"])
@pytest.mark.parametrize("tname", ["opaque", "ramp"])
def test_scenes(vs, scenes, scene, tname):
    v = vs.Volume.from_u8(scenes[f"{scene}_u8"])
    b = vs.classify(v, vs.TransferFunction(scenes[f"{scene}_{tname}_lut"]), dilate=True)
    _structures(vs, scenes, f"{scene}_{tname}_", b)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("name", list(KD_PARAMS))
def test_random_vs_oracle(vs, seed, name):
    rng = np.random.default_rng(seed)
    dims = tuple(int(d) for d in rng.integers(20, 70, size=3))
    coarse = rng.random((dims[0] // 6 + 1, dims[1] // 6 + 1, dims[2] // 6 + 1)) < 0.15
    bits = np.repeat(np.repeat(np.repeat(coarse, 6, 0), 6, 1), 6, 2)[:dims[0], :dims[1], :dims[2]]
    bits = bits & (rng.random(dims) < 0.6)
    b = vs.BinaryVolume(bits)
    t = vs.build_kdtree(vs.build_svt_grid(b), vs.BuildParams(**KD_PARAMS[name]))
    _check_tree(t, O.kd_build(bits, **KD_PARAMS[name]), name)


def test_box_queries(vs, rng):
    bits = rng.random((40, 33, 29)) < 0.01
    b = vs.BinaryVolume(bits)
    for bs in (8, 32):
        g = vs.build_svt_grid(b, bs)
        t = O.svt_build(bits, bs)
        for _ in range(25):
            lo = rng.integers(0, 30, size=3)
            hi = lo + rng.integers(1, 20, size=3)
            box = vs.Aabb(tuple(lo), tuple(hi))
            assert vs.box_count(g, box) == O.box_count(t, bits.shape, bs, lo, hi)
            got = vs.shrink_to_occupied(g, box)
            want = O.shrink_svt(t, bits.shape, bs, lo, hi)
            assert (got is None and want is None) or (got.lo, got.hi) == want


def test_index_kinds_and_render(vs, blobs64):
    """build_index for the table kinds == golden; frames through them == golden pixels."""
    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    b = vs.classify(v, tf, dilate=True)
    cam = vs.Camera(eye=tuple(blobs64["cam_eye"]), direction=tuple(blobs64["cam_dir"]),
                    up=tuple(blobs64["cam_up"]), extent=float(blobs64["cam_extent"]), width=96,
                    height=64)
    for kind in ("kd-shallow", "kd-deep-mls32", "kd-binned-mls32", "hybrid"):
        idx = vs.build_index(kind, b)
        tree = idx.tree if kind == "hybrid" else idx
        _check_tree(tree, _gold_tree(blobs64, "ramp03_" + ("kd-shallow" if kind == "hybrid" else kind)), kind)
        st = vs.report_stats(idx)
        assert st == {"node_count": tree.node_count, "height": tree.height()}
        rgba, samples = vs.render_float(v, tf, idx, cam)
        np.testing.assert_array_equal(samples, blobs64[f"ramp03_render_{kind}_samples"])
        np.testing.assert_array_equal(rgba, blobs64[f"ramp03_render_{kind}_rgba"])


def test_empty_and_dense(vs):
    z = vs.BinaryVolume(np.zeros((16, 16, 16), bool))
    t = vs.build_kdtree(vs.build_svt_grid(z))
    assert t.node_count == 0 and t.root == -1 and t.height() == 0
    d = vs.BinaryVolume(np.ones((24, 24, 24), bool))  # test_acceptance.py:116-124
    t = vs.build_kdtree(vs.build_svt_grid(d), vs.BuildParams(mode="deep"))
    assert t.node_count == 1 and t.height() == 1


@pytest.mark.parametrize("case", ["rand_64x48x40", "blocky48", "sparse64"])
def test_precompute_cell_boxes(vs, bitcases, case):
    dims = tuple(int(d) for d in bitcases[f"{case}_dims"])
    b = vs.BinaryVolume(unpack_bits(bitcases[f"{case}_bits"], dims))
    cells = vs.precompute_cell_boxes(b, 8)
    for f in ("codes", "coords", "lo", "hi", "occupied"):
        np.testing.assert_array_equal(getattr(cells, f), bitcases[f"{case}_cells8_{f}"], err_msg=f)


@pytest.mark.parametrize("dims,cs", [((37, 29, 45), 8), ((16, 8, 96), 8), ((70, 9, 1030), 8),
                                     ((33, 20, 41), 5), ((40, 40, 40), 16)])
def test_cell_boxes_ragged_vs_oracle(vs, rng, dims, cs):
    """k_cell_boxes8 (cs 8: warp per cell column, byte masks) and the generic per-cell kernel
    on ragged dims (partial cells on every axis, nz past one 32-word chunk) vs the oracle."""
    bits = rng.random(dims) < 0.004
    bits[:, :, -1] |= rng.random(dims[:2]) < 0.05  # flags in the last (partial) z word
    cells = vs.precompute_cell_boxes(vs.BinaryVolume(bits), cs)
    want = O.cell_boxes(bits, cs)
    for f in ("codes", "coords", "lo", "hi", "occupied"):
        np.testing.assert_array_equal(getattr(cells, f), want[f], err_msg=f)


def test_best_plane_apis_vs_reference_semantics(vs, rng):
    """sweep_best_plane / binned_best_plane on random boxes: the split the k-d builder takes
    at a root equals the single-box search, and the two-cluster known answer
    (test_kdtree.py:112-122, 217-231) holds."""
    bits = np.zeros((64, 24, 24), bool)
    bits[8:16, 8:16, 8:16] = True
    bits[40:48, 8:16, 8:16] = True
    b = vs.BinaryVolume(bits)
    g = vs.build_svt_grid(b)
    full = vs.Aabb((0, 0, 0), bits.shape)
    p = vs.sweep_best_plane(g, full)
    assert p is not None and p.axis == 0 and 16 <= p.position <= 40 and p.cost == 2 * 512
    cells = vs.precompute_cell_boxes(b, 8)
    pb = vs.binned_best_plane(cells, full)
    assert pb is not None and pb.axis == 0 and pb.cost == 2 * 512
    assert vs.sweep_best_plane(g, vs.Aabb((0, 0, 0), (4, 4, 4))) is None
    # a box inside one cluster: no cut beats its tight volume
    assert vs.sweep_best_plane(g, vs.Aabb((8, 8, 8), (16, 16, 16))) is None
    # random: the root decision of a deep sweep tree equals the single-box search
    for seed in range(4):
        r = np.random.default_rng(seed)
        bb = r.random((30, 26, 22)) < 0.03
        bv = vs.BinaryVolume(bb)
        gg = vs.build_svt_grid(bv)
        t = vs.build_kdtree(gg, vs.BuildParams(mode="deep"))
        if t.node_count > 1 and t.axis[0] >= 0:
            root = vs.Aabb(tuple(t.lo[0]), tuple(t.hi[0]))
            sp = vs.sweep_best_plane(gg, root)
            assert sp is not None and (sp.axis, sp.position) == (int(t.axis[0]), int(t.plane[0]))


def _blobby(rng, dims, dens, nbox):
    bits = rng.random(dims) < dens
    for _ in range(nbox):
        c = rng.integers(0, dims)
        r = rng.integers(2, 9, size=3)
        bits[tuple(slice(max(0, c[k] - r[k]), c[k] + r[k]) for k in range(3))] = True
    return bits


@pytest.mark.parametrize("name", ["kd-shallow", "kd-deep-mls32", "kd-binned-mls32", "kd-deep"])
def test_large_chunked_vs_oracle(vs, name):
    """Boxes wider than one 64-row span chunk / 1024-cell slab chunk (the atomic-merge paths of
    the span and cell-slab passes) and unaligned z ranges, against the oracle."""
    rng = np.random.default_rng(11)
    bits = _blobby(rng, (96, 272, 272), 0.0004, 40)
    t = vs.build_kdtree(vs.build_svt_grid(vs.BinaryVolume(bits)), vs.BuildParams(**KD_PARAMS[name]))
    _check_tree(t, O.kd_build(bits, **KD_PARAMS[name]), name)


@pytest.mark.parametrize("name", ["kd-deep-mls32", "kd-binned-mls32"])
def test_wide_levels_vs_oracle(vs, name):
    """Levels of thousands of nodes (multi-tile device scans) and > 64K rows (the per-level
    subtree-size / preorder finalisation), against the oracle."""
    rng = np.random.default_rng(7)
    bits = rng.random((320, 288, 256)) < 0.008
    t = vs.build_kdtree(vs.build_svt_grid(vs.BinaryVolume(bits)), vs.BuildParams(**KD_PARAMS[name]))
    want = O.kd_build(bits, **KD_PARAMS[name])
    assert len(want["axis"]) > 65536
    _check_tree(t, want, name)
