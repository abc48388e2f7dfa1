"""Multi-channel volumes (configs[4]) on the GPU: exact reduction to the reference's
single-channel frames, and 4-channel frames vs the C restatement (oracle.render_multi)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    return vs


def _cam(vs, g, w, h):
    return vs.Camera(eye=tuple(g["cam_eye"]), direction=tuple(g["cam_dir"]), up=tuple(g["cam_up"]),
                     extent=float(g["cam_extent"]), width=w, height=h)


def test_reduces_to_single_channel(vs, blobs64):
    from paper_1912_09596_b200.multichannel import classify_multi, render_float_multi

    u8 = blobs64["u8"]
    vols = [vs.Volume.from_u8(u8), vs.Volume.from_u8(u8[::-1].copy()), vs.Volume.from_u8(u8.T.copy())]
    zero = vs.TransferFunction(np.zeros((256, 4), np.float32))
    tfs = [vs.TransferFunction(blobs64["ramp03_lut"]), zero, zero]
    b = classify_multi(vols, tfs, dilate=True)
    idx = vs.build_index("lbvh", b)
    single = vs.build_index("lbvh", vs.classify(vols[0], tfs[0], dilate=True))
    np.testing.assert_array_equal(idx.lo, single.lo)
    cam = _cam(vs, blobs64, 96, 64)
    rgba, samples = render_float_multi(vols, tfs, idx, cam)
    np.testing.assert_array_equal(samples, blobs64["ramp03_render_lbvh_samples"])
    np.testing.assert_array_equal(rgba, blobs64["ramp03_render_lbvh_rgba"])


@pytest.mark.parametrize("kind", ["naive", "grid", "lbvh"])
def test_four_channels_vs_restatement(vs, blobs64, kind):
    from paper_1912_09596_b200.multichannel import classify_multi, render_float_multi

    u8 = blobs64["u8"]
    chans = [u8, np.ascontiguousarray(u8[::-1]), np.ascontiguousarray(u8.transpose(1, 0, 2)),
             np.ascontiguousarray(u8[:, ::-1])]
    luts = []
    for c, t in enumerate((0.3, 0.4, 0.5, 0.6)):
        lut = vs.TransferFunction.ramp(t).lut.copy()
        lut[:, c % 3] = 0.9
        luts.append(lut)
    vols = [vs.Volume.from_u8(c) for c in chans]
    tfs = [vs.TransferFunction(l) for l in luts]
    b = classify_multi(vols, tfs, dilate=True)
    # union classification == OR of the per-channel oracle classifications, dilated
    plain = np.zeros(u8.shape, bool)
    for c, l in zip(chans, luts):
        plain |= O.classify(c, l, dilate=False)[0]
    np.testing.assert_array_equal(classify_multi(vols, tfs, dilate=False).bits, plain)
    idx = vs.build_index(kind, b)
    cam = _cam(vs, blobs64, 96, 64)
    rgba, samples = render_float_multi(vols, tfs, idx, cam)
    if kind == "naive":
        oidx = None
    elif kind == "grid":
        oidx = {"occupied": idx.occupied, "cell_size": 16}
    else:
        oidx = {"lo": idx.lo, "hi": idx.hi, "left": idx.left, "right": idx.right,
                "root": idx.root, "height": idx.height()}
    orgba, osamples = O.render_multi(kind, chans, luts, oidx, cam)
    np.testing.assert_array_equal(samples, osamples)
    assert float(np.max(np.abs(rgba - orgba))) <= 1e-3
    np.testing.assert_array_equal(rgba, orgba)


@pytest.mark.parametrize("nch", [1, 2])
def test_channel_counts_vs_restatement(vs, blobs64, nch):
    """1 and 2 channels (the 1- and 2-word interleaved gather layouts) vs the restatement."""
    from paper_1912_09596_b200.multichannel import classify_multi, render_float_multi

    u8 = blobs64["u8"]
    chans = [u8, np.ascontiguousarray(u8[::-1])][:nch]
    luts = []
    for c, t in enumerate((0.3, 0.45)[:nch]):
        lut = vs.TransferFunction.ramp(t).lut.copy()
        lut[:, c] = 0.8
        luts.append(lut)
    vols = [vs.Volume.from_u8(c) for c in chans]
    tfs = [vs.TransferFunction(l) for l in luts]
    idx = vs.build_index("lbvh", classify_multi(vols, tfs, dilate=True))
    cam = _cam(vs, blobs64, 80, 56)
    rgba, samples = render_float_multi(vols, tfs, idx, cam)
    oidx = {"lo": idx.lo, "hi": idx.hi, "left": idx.left, "right": idx.right,
            "root": idx.root, "height": idx.height()}
    orgba, osamples = O.render_multi("lbvh", chans, luts, oidx, cam)
    np.testing.assert_array_equal(samples, osamples)
    np.testing.assert_array_equal(rgba, orgba)


def test_tile_frame_multi_async(vs, blobs64):
    """TileRenderer.frame_multi_async == render_frame_multi (pixels and sample count)."""
    from paper_1912_09596_b200.multichannel import classify_multi, render_frame_multi
    from paper_1912_09596_b200.tiles import TileRenderer

    u8 = blobs64["u8"]
    vols = [vs.Volume.from_u8(u8), vs.Volume.from_u8(np.ascontiguousarray(u8[::-1]))]
    tfs = [vs.TransferFunction.ramp(0.3), vs.TransferFunction.ramp(0.5)]
    idx = vs.build_index("lbvh", classify_multi(vols, tfs, dilate=True))
    cam = _cam(vs, blobs64, 72, 40)
    ref = render_frame_multi(vols, tfs, idx, cam)
    fr = TileRenderer(cam.width, cam.height).frame_multi_async(vols, tfs, idx, cam).result()
    np.testing.assert_array_equal(fr.pixels, ref.pixels)
    assert fr.sample_count == ref.sample_count


@pytest.mark.parametrize("nch", [2, 4])
def test_smooth_channels_band_tfs_vs_restatement(vs, nch):
    """Smooth fields (many interpolated values near bin edges: the FP32 bin filter's fallback
    path) with narrow-band TFs, 2 and 4 channels, against the restatement bit for bit."""
    from paper_1912_09596_b200.multichannel import classify_multi, render_float_multi

    n = 36
    g = np.mgrid[0:n, 0:n, 0:n].astype(np.float64)
    chans, luts = [], []
    for c in range(nch):
        f = 0.5 + 0.5 * np.sin(g[0] / (4.0 + c)) * np.cos(g[1] / (6.0 - c * 0.5)) * \
            np.sin(g[2] / 3.0 + c)
        chans.append(np.clip(np.rint(f * 255.0), 0, 255).astype(np.uint8))
        lut = np.zeros((256, 4), dtype=np.float32)
        lut[:, c % 3] = 0.9
        lut[90 + 30 * c:93 + 30 * c, 3] = 0.5   # narrow band per channel
        lut[200:, 3] = 0.2
        luts.append(lut)
    vols = [vs.Volume.from_u8(u) for u in chans]
    tfs = [vs.TransferFunction(l) for l in luts]
    idx = vs.build_index("lbvh", classify_multi(vols, tfs, dilate=True))
    cam = vs.Camera.orbit((n, n, n), 41.0, 23.0, width=64, height=48)
    rgba, samples = render_float_multi(vols, tfs, idx, cam)
    oidx = {"lo": idx.lo, "hi": idx.hi, "left": idx.left, "right": idx.right,
            "root": idx.root, "height": idx.height()}
    orgba, osamples = O.render_multi("lbvh", chans, luts, oidx, cam)
    np.testing.assert_array_equal(samples, osamples)
    np.testing.assert_array_equal(rgba, orgba)
