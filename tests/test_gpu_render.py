"""GPU parity of the ray marcher (csrc/render.cu) against the reference's golden frames and the
CPU oracle: float RGBA and per-pixel sample counts are compared EXACTLY (the north-star bound
is max-abs 1e-3 per channel; the FP64 path reproduces the reference bit for bit, so the test
asserts equality and reports the max-abs difference on failure)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
RGBA_TOL = 1e-3  # BASELINE.json north_star: rendered RGBA within max-abs 1e-3 per channel


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    return vs


def _cam_from(vs, g, w, h):
    return vs.Camera(eye=tuple(g["cam_eye"]), direction=tuple(g["cam_dir"]), up=tuple(g["cam_up"]),
                     extent=float(g["cam_extent"]), width=w, height=h)


def _kd(vs, g, p, dims):
    return vs.KdTree(g[f"{p}_lo"], g[f"{p}_hi"], g[f"{p}_axis"], g[f"{p}_plane"], g[f"{p}_left"],
                     g[f"{p}_right"], int(g[f"{p}_root"]), dims)


def _index(vs, kind, g, prefix, v, tf):
    dims = v.dims
    b = vs.classify(v, tf, dilate=True)
    if kind == "naive":
        return None
    if kind == "grid":
        return vs.build_index("grid", b)
    if kind == "lbvh":
        return vs.build_index("lbvh", b)
    if kind == "hybrid":
        return vs.HybridGrid(_kd(vs, g, prefix + "kd-shallow", dims), vs.build_index("grid", b))
    return _kd(vs, g, prefix + kind, dims)


def _assert_rgba(got, want):
    diff = float(np.max(np.abs(got - want))) if got.size else 0.0
    assert diff <= RGBA_TOL, diff
    np.testing.assert_array_equal(got, want, err_msg=f"max-abs {diff:g}")


@pytest.mark.parametrize("tname", ["ramp03", "band"])
@pytest.mark.parametrize("kind", ["naive", "grid", "lbvh", "kd-shallow", "kd-deep-mls32",
                                  "kd-binned-mls32", "hybrid"])
def test_blobs64_render_exact(vs, blobs64, tname, kind):
    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64[f"{tname}_lut"])
    idx = _index(vs, kind, blobs64, f"{tname}_", v, tf)
    cam = _cam_from(vs, blobs64, 96, 64)
    rgba, samples = vs.render_float(v, tf, idx, cam)
    np.testing.assert_array_equal(samples, blobs64[f"{tname}_render_{kind}_samples"])
    _assert_rgba(rgba, blobs64[f"{tname}_render_{kind}_rgba"])
    fr = vs.render_frame(v, tf, idx, cam)
    np.testing.assert_array_equal(fr.pixels, blobs64[f"{tname}_render_{kind}_pixels"])
    assert fr.sample_count == int(blobs64[f"{tname}_render_{kind}_samples"].sum())


@pytest.mark.parametrize("scene", ["shell", "menger"])
@pytest.mark.parametrize("tname", ["opaque", "ramp"])
def test_scene_frames(vs, scenes, scene, tname):
    u8 = scenes[f"{scene}_u8"]
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction(scenes[f"{scene}_{tname}_lut"])
    cam = vs.Camera.orbit(u8.shape, 25.0, 20.0, width=64)
    for kind in ("naive", "grid", "lbvh", "kd-deep-mls32", "hybrid"):
        idx = _index(vs, kind, scenes, f"{scene}_{tname}_", v, tf)
        fr = vs.render_frame(v, tf, idx, cam)
        np.testing.assert_array_equal(fr.pixels, scenes[f"{scene}_{tname}_render_{kind}_pixels"],
                                      err_msg=kind)
        assert fr.sample_count == int(scenes[f"{scene}_{tname}_render_{kind}_samples"]), kind
    if tname == "ramp":
        fr = vs.render_frame(v, tf, None, cam, interp="nearest")
        np.testing.assert_array_equal(fr.pixels, scenes[f"{scene}_ramp_render_nearest_pixels"])
        assert fr.sample_count == int(scenes[f"{scene}_ramp_render_nearest_samples"])


def test_float_volume_render(vs, misc):
    data, lut = misc["f32_data"], misc["f32_lut"]
    v = vs.Volume(data)
    tf = vs.TransferFunction(lut)
    b = vs.classify(v, tf, dilate=True)
    cam = vs.Camera.orbit(data.shape, 40.0, -20.0, width=32, height=24)
    dil, _ = O.classify(data, lut, dilate=True)
    kd = O.kd_build(dil, mode="deep")
    kdt = vs.KdTree(kd["lo"], kd["hi"], kd["axis"], kd["plane"], kd["left"], kd["right"],
                    kd["root"], data.shape)
    for kind, idx in (("naive", None), ("lbvh", vs.build_index("lbvh", b)), ("kd", kdt)):
        rgba, samples = vs.render_float(v, tf, idx, cam)
        np.testing.assert_array_equal(samples, misc[f"f32_render_{kind}_samples"])
        _assert_rgba(rgba, misc[f"f32_render_{kind}_rgba"])


def test_single_ray_api(vs, blobs64):
    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    dims = v.dims
    idxs = {"naive": None, "grid": _index(vs, "grid", blobs64, "ramp03_", v, tf),
            "lbvh": _index(vs, "lbvh", blobs64, "ramp03_", v, tf),
            "kd": _index(vs, "kd-deep-mls32", blobs64, "ramp03_", v, tf),
            "hybrid": _index(vs, "hybrid", blobs64, "ramp03_", v, tf)}
    fns = {"naive": lambda r, i: vs.traverse_naive(r, dims), "grid": vs.traverse_grid,
           "lbvh": vs.traverse_lbvh, "kd": vs.traverse_kd, "hybrid": vs.traverse_hybrid}
    for kind, idx in idxs.items():
        counts = blobs64[f"trav_{kind}_counts"]
        segs = blobs64[f"trav_{kind}_segs"]
        off = 0
        for o, d, c in zip(blobs64["rays_o"], blobs64["rays_d"], counts):
            got = fns[kind](vs.Ray(tuple(o), tuple(d)), idx)
            np.testing.assert_array_equal(got.t, segs[off:off + c], err_msg=kind)
            off += c
    for r, (o, d) in enumerate(zip(blobs64["rays_o"], blobs64["rays_d"])):
        ray = vs.Ray(tuple(o), tuple(d))
        segs = vs.traverse_naive(ray, dims)
        np.testing.assert_array_equal(vs.integrate(ray, segs, v, tf), blobs64["integrate_rgba"][r])
        assert vs.sample_count_of(ray, segs, dims) == int(blobs64["integrate_samples"][r])


@pytest.mark.parametrize("az,el", [(0.0, 0.0), (90.0, 0.0), (180.0, 89.9), (33.0, -47.0)])
def test_axis_aligned_and_oblique_vs_oracle(vs, blobs64, az, el):
    """Zero direction components (containment slabs, R_FAR crossings) and steep views."""
    u8 = blobs64["u8"]
    lut = blobs64["ramp03_lut"]
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction(lut)
    cam = vs.Camera.orbit(u8.shape, az, el, width=48, height=40)
    b = vs.classify(v, tf, dilate=True)
    grid = vs.build_index("grid", b)
    lbvh = vs.build_index("lbvh", b)
    for kind, idx, oidx in (("naive", None, None),
                            ("grid", grid, {"occupied": grid.occupied, "cell_size": 16}),
                            ("lbvh", lbvh, {"lo": lbvh.lo, "hi": lbvh.hi, "left": lbvh.left,
                                            "right": lbvh.right, "root": lbvh.root,
                                            "height": lbvh.height()})):
        rgba, samples = vs.render_float(v, tf, idx, cam)
        orgba, osamples = O.render(kind, u8, lut, oidx, cam, nthreads=4)
        np.testing.assert_array_equal(samples, osamples, err_msg=kind)
        _assert_rgba(rgba, orgba)


def test_row_stripes_assemble(vs, blobs64):
    """Interleaved row stripes (the multi-GPU tile split) reassemble the full frame."""
    import torch

    from paper_1912_09596_b200.render import RenderTarget, RowsDesc, render_rows

    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=40, height=37)
    full = vs.render_frame(v, tf, idx, cam)
    for nparts, stripe in ((2, 8), (3, 4), (4, 1)):
        img = np.zeros_like(full.pixels)
        total = 0
        for part in range(nparts):
            rows = [j for j in range(cam.height) if (j // stripe) % nparts == part]
            tgt = RenderTarget(cam.width, len(rows))
            render_rows(v, tf, idx, cam, tgt, rows=RowsDesc(len(rows), stripe, nparts, part))
            img[rows] = tgt.rgba8.cpu().numpy()
            total += int(tgt.total.item())
        np.testing.assert_array_equal(img, full.pixels)
        assert total == full.sample_count
    torch.cuda.synchronize()


def test_render_errors(vs, blobs64):
    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    cam = vs.Camera.orbit(v.dims, 0.0, width=8)
    with pytest.raises(ValueError):
        vs.render_frame(v, tf, None, cam, dt=0.0)
    with pytest.raises(ValueError):
        vs.render_frame(v, tf, None, cam, interp="cubic")
    # zero-alpha TF: nothing visible, samples still counted on the naive lattice
    empty = vs.TransferFunction(np.zeros((256, 4), np.float32))
    fr = vs.render_frame(v, empty, None, cam)
    assert fr.pixels.max() == 0 and fr.sample_count > 0
    lb = vs.build_index("lbvh", vs.classify(v, empty, dilate=True))
    assert vs.render_frame(v, empty, lb, cam).sample_count == 0


@pytest.mark.parametrize("az,el", [(30.0, 15.0), (0.0, 0.0), (90.0, 0.0), (200.0, -35.0),
                                   (45.0, 45.0)])
def test_lbvh_brick_dda_equals_tree_walk(vs, az, el):
    """The brick-DDA leaf enumeration and the reference's tree walk give identical frames,
    on a volume whose dims are not brick multiples (clipped border bricks)."""
    from paper_1912_09596_b200.render import RenderTarget, index_desc, render_rows

    rng = np.random.default_rng(7)
    dims = (45, 38, 52)
    coarse = rng.integers(0, 256, size=(10, 10, 11), dtype=np.uint8)
    u8 = np.repeat(np.repeat(np.repeat(coarse, 5, 0), 4, 1), 5, 2)[:dims[0], :dims[1], :dims[2]].copy()
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(0.7)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    cam = vs.Camera.orbit(dims, az, el, width=57, height=43)
    outs = []
    for dda in (False, True):
        tgt = RenderTarget(cam.width, cam.height, want_rgba64=True, want_samples=True)
        render_rows(v, tf, idx, cam, tgt, idx_desc=index_desc(idx, use_brick_dda=dda))
        outs.append((tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy(), int(tgt.flags.item())))
    assert outs[0][2] == 0 and outs[1][2] == 0
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    lb = {"lo": idx.lo, "hi": idx.hi, "left": idx.left, "right": idx.right, "root": idx.root,
          "height": idx.height()}
    orgba, osamples = O.render("lbvh", u8, tf.lut, lb, cam, nthreads=4)
    np.testing.assert_array_equal(outs[1][1], osamples)
    np.testing.assert_array_equal(outs[1][0], orgba)


@pytest.mark.parametrize("az,el", [(0.0, 0.0), (90.0, 0.0), (123.0, 37.0), (300.0, -60.0)])
def test_quad_gather_equals_byte_gather(vs, az, el):
    """The packed (y,z) 2x2 trilinear gather gives the same frames as eight byte loads,
    including the clamped borders (every face of a small volume is crossed)."""
    from paper_1912_09596_b200.render import RenderTarget, render_rows, volume_desc

    rng = np.random.default_rng(11)
    u8 = rng.integers(0, 256, size=(13, 17, 11), dtype=np.uint8)
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(0.2)
    cam = vs.Camera.orbit(u8.shape, az, el, width=40, height=33, zoom=1.3)
    outs = []
    for q in (False, True):
        tgt = RenderTarget(cam.width, cam.height, want_rgba64=True, want_samples=True)
        render_rows(v, tf, None, cam, tgt, vol_desc=volume_desc(v, quads=q))
        outs.append((tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    orgba, osamples = O.render("naive", u8, tf.lut, None, cam, nthreads=4)
    np.testing.assert_array_equal(outs[1][0], orgba)


@pytest.mark.parametrize("kind", ["naive", "grid", "lbvh", "kd-deep-mls32", "hybrid"])
def test_two_phase_equals_fused(vs, blobs64, kind):
    """Two-phase rendering (segment buffer, incl. overflow re-traversal at cap 1) == fused."""
    from paper_1912_09596_b200.render import RenderTarget, render_rows

    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    idx = _index(vs, kind, blobs64, "ramp03_", v, tf)
    cam = _cam_from(vs, blobs64, 96, 64)
    outs = []
    for cap in (0, 1, 16):
        tgt = RenderTarget(cam.width, cam.height, want_rgba64=True, want_samples=True, seg_cap=cap)
        render_rows(v, tf, idx, cam, tgt)
        outs.append((tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy()))
    for o in outs[1:]:
        np.testing.assert_array_equal(o[1], outs[0][1])
        np.testing.assert_array_equal(o[0], outs[0][0])
    np.testing.assert_array_equal(outs[0][1], blobs64[f"ramp03_render_{kind}_samples"])


def test_u8_table_option_equal(vs, blobs64):
    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    cam = _cam_from(vs, blobs64, 96, 64)
    outs = [vs.render_float(v, tf, None, cam, flags=f) for f in (0, 1)]
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[1][0], blobs64["ramp03_render_naive_rgba"])


@pytest.mark.parametrize("kind", ["naive", "grid", "lbvh", "kd-deep-mls32", "hybrid"])
def test_persistent_two_phase_equal(vs, blobs64, kind):
    """Persistent-lane two-phase rendering (render option bit 1) == fused, incl. overflow."""
    from paper_1912_09596_b200 import _lib
    from paper_1912_09596_b200.render import RenderTarget, render_rows

    v = vs.Volume.from_u8(blobs64["u8"])
    tf = vs.TransferFunction(blobs64["ramp03_lut"])
    idx = _index(vs, kind, blobs64, "ramp03_", v, tf)
    cam = _cam_from(vs, blobs64, 96, 64)
    outs = []
    for opts, cap in ((1, 0), (3, 1), (3, 32), (5, 1), (5, 32)):
        tgt = RenderTarget(cam.width, cam.height, want_rgba64=True, want_samples=True,
                           seg_cap=cap)
        render_rows(v, tf, idx, cam, tgt, flags=opts)
        outs.append((tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy(),
                     int(tgt.total.item())))
    for o in outs[1:]:
        np.testing.assert_array_equal(o[1], outs[0][1])
        np.testing.assert_array_equal(o[0], outs[0][0])
        assert o[2] == outs[0][2]


def test_tile_frame_pinned_buffers(vs, blobs64):
    """TileRenderer.frame hands out pinned pixel buffers: a held Frame is never overwritten,
    a dropped one is recycled; pixels and sample counts equal render_frame's."""
    from paper_1912_09596_b200.tiles import TileRenderer

    v = vs.Volume.from_u8(blobs64["u8"])
    tfs = [vs.TransferFunction.ramp(0.3), vs.TransferFunction.ramp(0.6)]
    cam = _cam_from(vs, blobs64, 80, 48)
    tr = TileRenderer(cam.width, cam.height)
    refs = []
    for tf in tfs:
        idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
        refs.append(vs.render_frame(v, tf, idx, cam))
    idx0 = vs.build_index("lbvh", vs.classify(v, tfs[0], dilate=True))
    idx1 = vs.build_index("lbvh", vs.classify(v, tfs[1], dilate=True))
    f0 = tr.frame(v, tfs[0], idx0, cam)
    keep = f0.pixels.copy()
    f1 = tr.frame(v, tfs[1], idx1, cam)
    np.testing.assert_array_equal(f0.pixels, keep)          # still held: not overwritten
    np.testing.assert_array_equal(f0.pixels, refs[0].pixels)
    np.testing.assert_array_equal(f1.pixels, refs[1].pixels)
    assert (f0.sample_count, f1.sample_count) == (refs[0].sample_count, refs[1].sample_count)
    assert len(tr._pinned_ring) == 2
    del f0
    f2 = tr.frame(v, tfs[0], idx0, cam)                       # reuses the dropped buffer
    assert len(tr._pinned_ring) == 2
    np.testing.assert_array_equal(f2.pixels, refs[0].pixels)
    # pipelined readback: frame k+1 is queued before frame k is collected
    p0 = tr.frame_async(v, tfs[1], idx1, cam)
    p1 = tr.frame_async(v, tfs[0], idx0, cam)
    g0, g1 = p0.result(), p1.result()
    np.testing.assert_array_equal(g0.pixels, refs[1].pixels)
    np.testing.assert_array_equal(g1.pixels, refs[0].pixels)
    assert (g0.sample_count, g1.sample_count) == (refs[1].sample_count, refs[0].sample_count)


@pytest.mark.parametrize("kind", ["lbvh", "grid"])
def test_configs1_row_band_vs_oracle(vs, kind):
    """BASELINE configs[1] scale (256^3 blobs, 1024x1024): a 16-row band through the middle of
    the GPU frame equals the oracle's render of the same rows, float RGBA and sample counts."""
    from paper_1912_09596_b200.synth import gen_blobs_u8

    u8_dev = gen_blobs_u8((256, 256, 256), 400, seed=7, sigma=3.0)
    u8 = u8_dev.cpu().numpy()
    v = vs.Volume.from_u8(u8_dev)
    tf = vs.TransferFunction.ramp(0.3)
    idx = vs.build_index(kind, vs.classify(v, tf, dilate=True))
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1024, height=1024)
    rgba, samples = vs.render_float(v, tf, idx, cam)
    if kind == "lbvh":
        oidx = {"lo": idx.lo, "hi": idx.hi, "left": idx.left, "right": idx.right,
                "root": idx.root, "height": idx.height()}
    else:
        oidx = {"occupied": idx.occupied, "cell_size": 16}
    r0, r1 = 504, 520
    orgba, osamples = O.render(kind, u8, tf.lut, oidx, cam, rows=(r0, r1), nthreads=8)
    np.testing.assert_array_equal(samples[r0:r1].reshape(-1), osamples.reshape(-1))
    np.testing.assert_array_equal(rgba[r0:r1].reshape(-1, 4), orgba.reshape(-1, 4))


@pytest.mark.parametrize("kind", ["naive", "lbvh", "kd-deep-mls32"])
@pytest.mark.parametrize("seg_cap", [0, 16])
def test_early_ray_termination_bound(vs, blobs64, kind, seg_cap):
    """ERT at eps: every float RGBA channel within eps of the full (reference) integral, never
    more samples; eps = 0 is the reference integrator bit for bit."""
    from paper_1912_09596_b200.render import RenderTarget, render_rows

    v = vs.Volume.from_u8(blobs64["u8"])
    lut = vs.TransferFunction.ramp(0.05).lut.copy()
    lut[:, 3] = np.minimum(1.0, lut[:, 3] * 4.0)   # dense, opaque: many rays saturate
    tf = vs.TransferFunction(lut)
    idx = vs.build_index(kind, vs.classify(v, tf, dilate=True))
    cam = _cam_from(vs, blobs64, 96, 64)
    outs = {}
    for eps in (0.0, 1e-3, 1e-2):
        tgt = RenderTarget(cam.width, cam.height, want_rgba64=True, want_samples=True,
                           seg_cap=seg_cap)
        render_rows(v, tf, idx, cam, tgt, ert_eps=eps)
        outs[eps] = (tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy())
    full, fs = outs[0.0]
    orgba, osamples = vs.render_float(v, tf, idx, cam)
    np.testing.assert_array_equal(full, orgba)
    np.testing.assert_array_equal(fs, osamples)
    assert float((full[..., 3] >= 1 - 1e-2).mean()) > 0.1  # the case exercises termination
    for eps in (1e-3, 1e-2):
        rgba, s = outs[eps]
        assert float(np.max(np.abs(rgba - full))) <= eps
        assert np.all(s <= fs) and int(s.sum()) < int(fs.sum())


@pytest.mark.parametrize("dims", [(100, 90, 70), (64, 64, 64)])
def test_brick_run_shortcut_equals_per_brick_slab(vs, dims):
    """k_segments_brick's run shortcut (occupied interior bricks extend the merged run to the
    next crossing) == every brick through slab() == the generic generator kernel, at odd dims
    (clipped border bricks) and several views."""
    from paper_1912_09596_b200 import _lib

    rng = np.random.default_rng(3)
    u8 = (rng.random(dims) * 255).astype(np.uint8)
    u8[rng.random(dims) < 0.7] = 0
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(0.5)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    for az, el in ((30.0, 15.0), (0.0, 0.0), (90.0, 45.0), (211.0, -33.0)):
        cam = vs.Camera.orbit(v.dims, az, el, width=120, height=96)
        outs = [vs.render_float(v, tf, idx, cam, flags=f) for f in (1, 1 | 16, 1 | 4)]
        for o in outs[1:]:
            np.testing.assert_array_equal(o[1], outs[0][1])
            np.testing.assert_array_equal(o[0], outs[0][0])


@pytest.mark.parametrize("kind", ["lbvh", "grid", "hybrid"])
def test_sign_specialised_traversal_all_octants(vs, kind):
    """The traversal kernels instantiated per sign pattern of the (frame-uniform) ray direction
    == the generic generator kernel, for all eight octants and an axis-aligned view (the
    general instantiation), at odd dims."""
    rng = np.random.default_rng(5)
    dims = (70, 53, 96)
    u8 = (rng.random(dims) * 255).astype(np.uint8)
    u8[rng.random(dims) < 0.8] = 0
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(0.5)
    idx = vs.build_index(kind, vs.classify(v, tf, dilate=True))
    views = [(az, el) for az in (45.0, 135.0, 225.0, 315.0) for el in (30.0, -30.0)]
    for az, el in views + [(90.0, 0.0)]:
        cam = vs.Camera.orbit(v.dims, az, el, width=72, height=60)
        fast = vs.render_float(v, tf, idx, cam, flags=1)
        generic = vs.render_float(v, tf, idx, cam, flags=1 | 4)
        np.testing.assert_array_equal(fast[1], generic[1], err_msg=f"{kind} {az} {el}")
        np.testing.assert_array_equal(fast[0], generic[0], err_msg=f"{kind} {az} {el}")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["naive", "lbvh", "grid", "hybrid"])
def test_fp32_bin_filter_equals_fp64_bins(vs, kind):
    """The integration kernel's FP32 bin filter (FP64 only within 1e-3 of a bin edge) gives
    the reference's bins: frames and sample counts bit-equal to every sample in FP64, for a
    smooth volume (many interpolated values near bin edges), ramp and band TFs."""
    from paper_1912_09596_b200 import _lib

    n = 40
    g = np.mgrid[0:n, 0:n, 0:n].astype(np.float64)
    field = 0.5 + 0.5 * np.sin(g[0] / 5.0) * np.cos(g[1] / 7.0) * np.sin(g[2] / 3.0 + 1.0)
    u8 = np.clip(np.rint(field * 255.0), 0, 255).astype(np.uint8)
    v = vs.Volume.from_u8(u8)
    lut = np.zeros((256, 4), dtype=np.float32)
    lut[:, :3] = np.linspace(0, 1, 256)[:, None]
    lut[100:103, 3] = 0.6   # narrow band: bins decided right at the edges matter
    lut[180:, 3] = 0.3
    tfs = [vs.TransferFunction.ramp(0.45), vs.TransferFunction(lut)]
    for tf in tfs:
        idx = None if kind == "naive" else vs.build_index(kind, vs.classify(v, tf, dilate=True))
        for az, el in ((30.0, 15.0), (123.0, -40.0)):
            cam = vs.Camera.orbit(v.dims, az, el, width=96, height=80)
            fast = vs.render_float(v, tf, idx, cam, flags=1)
            exact = vs.render_float(v, tf, idx, cam, flags=1 | 2)
            np.testing.assert_array_equal(fast[1], exact[1])
            np.testing.assert_array_equal(fast[0], exact[0])
