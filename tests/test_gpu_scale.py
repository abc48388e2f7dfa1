"""Parity against the CPU oracle at the BASELINE configs' own sizes.

* configs[1] 256^3 (400 blobs): LBVH / grid / kd-shallow arrays and a frame.
* configs[2] 512^3 (3,200 blobs) x ramp t = 0.6 / 0.3 / 0.0: kd-deep-mls32, kd-deep-mls128 and
  kd-binned-mls32 arrays equal the oracle's; node counts and heights equal SURVEY App. B
  (the unmodified reference's numbers).
* configs[3] 1024^3 (25,600 blobs) x t = 0.6 / 0.3 / 0.0: LBVH, grid, kd-shallow and hybrid
  arrays equal the oracle's full-size builds; full 1920x1080 LBVH and hybrid frames (float
  RGBA and per-pixel samples) equal the oracle's at t = 0.3.
* configs[4] 4-channel 1024^3: the union LBVH equals the oracle's, and a 1920-wide row band of
  the 1080p frame equals the oracle's multi-channel restatement.

The oracle runs multi-threaded (classification, dilation, brick votes, rendering); a 1024^3
TF step takes seconds, so everything is compared outright -- bit-exact for bits, arrays and
counts, exact float RGBA (the 1e-3 RGBA tolerance of the north star holds with margin 0).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import KD_ARGS
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TREE = ("lo", "hi", "left", "right")
KD = TREE + ("axis", "plane")
LBVH = TREE + ("leaf_brick", "brick_coords")


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    O.set_threads(0)  # all host cores
    return vs


def _same(got, want: dict, fields, what):
    for f in fields:
        np.testing.assert_array_equal(getattr(got, f), want[f], err_msg=f"{what}.{f}")
    assert got.height() == want["height"], what


def _oracle_lbvh(bits):
    coords, codes = O.flag_bricks(bits, 8)
    return O.build_lbvh(coords, codes, 8, bits.shape)


def _blobs(n, nblobs, seed=7):
    from paper_1912_09596_b200.synth import gen_blobs_u8

    u8 = gen_blobs_u8((n, n, n), nblobs, seed=seed, sigma=3.0)
    return u8, u8.cpu().numpy()


# -- configs[1] ---------------------------------------------------------------------------------

def test_config1_256_vs_oracle(vs):
    u8, host = _blobs(256, 400)
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(0.3)
    b = vs.classify(v, tf, dilate=True)
    lb = vs.build_index("lbvh", b)
    assert lb.n_bricks == 3716 and lb.node_count == 7431 and lb.height() == 16
    bits, _ = O.classify(host, tf.lut, dilate=True)
    ref = _oracle_lbvh(bits)
    _same(lb, ref, LBVH, "lbvh")
    np.testing.assert_array_equal(vs.build_index("grid", b).occupied, O.macro_grid(bits, 16))
    _same(vs.build_index("kd-shallow", b), O.kd_build(bits, mode="shallow"), KD, "kd-shallow")
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1024, height=1024)
    rgba, samples = vs.render_float(v, tf, lb, cam)
    orgba, osamples = O.render("lbvh", host, tf.lut, ref, cam)
    assert int(samples.sum()) == 20328072  # the reference's frame sample count
    np.testing.assert_array_equal(samples, osamples)
    np.testing.assert_array_equal(rgba, orgba)


# -- configs[2] ---------------------------------------------------------------------------------

# SURVEY App. B (unmodified reference, same volume): (nodes, height) per t
APP_B_512 = {
    0.6: {"kd-deep-mls32": (11127, 82), "kd-binned-mls32": (10697, 24)},
    0.3: {"kd-deep-mls32": (41543, 62), "kd-deep-mls128": (41499, 62),
          "kd-binned-mls32": (24397, 26)},
    0.0: {"kd-deep-mls32": (149221, 63), "kd-deep-mls128": (62425, 53),
          "kd-binned-mls32": (83457, 27)},
}


@pytest.fixture(scope="module")
def vol512(vs):
    return _blobs(512, 3200)


@pytest.mark.parametrize("t", [0.6, 0.3, 0.0])
def test_config2_512_kd_trees_vs_oracle(vs, vol512, t):
    u8, host = vol512
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(t)
    b = vs.classify(v, tf, dilate=True)
    bits, _ = O.classify(host, tf.lut, dilate=True)
    np.testing.assert_array_equal(b.bits, bits)
    for kind in ("kd-deep-mls32", "kd-deep-mls128", "kd-binned-mls32"):
        kd = vs.build_index(kind, b)
        _same(kd, O.kd_build(bits, **KD_ARGS[kind]), KD, f"{kind}@{t}")
        if kind in APP_B_512[t]:
            assert (kd.node_count, kd.height()) == APP_B_512[t][kind], (kind, t)


# -- configs[3] ---------------------------------------------------------------------------------

@pytest.fixture(scope="module")
def vol1024(vs):
    return _blobs(1024, 25600)


_ORACLE_1024 = {}


@pytest.mark.parametrize("t", [0.6, 0.3, 0.0])
def test_config3_1024_indices_vs_oracle(vs, vol1024, t):
    u8, host = vol1024
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(t)
    b = vs.classify(v, tf, dilate=True)
    lb = vs.build_index("lbvh", b)
    grid = vs.build_index("grid", b)
    hyb = vs.build_index("hybrid", b)
    bits, plain = O.classify(host, tf.lut, dilate=True)
    assert vs.classify(v, tf).base_count() == plain
    ref = _oracle_lbvh(bits)
    _same(lb, ref, LBVH, f"lbvh@{t}")
    occ = O.macro_grid(bits, 16)
    np.testing.assert_array_equal(grid.occupied, occ)
    shallow = O.kd_build(bits, mode="shallow")
    _same(hyb.tree, shallow, KD, f"hybrid.tree@{t}")
    np.testing.assert_array_equal(hyb.grid.occupied, occ)
    _same(vs.build_index("kd-shallow", b), shallow, KD, f"kd-shallow@{t}")
    if t == 0.3:  # SURVEY App. B (reference): n_b 243,434, 486,867 nodes, height 22; (11, 6)
        assert (lb.n_bricks, lb.node_count, lb.height()) == (243434, 486867, 22)
        assert (hyb.tree.node_count, hyb.tree.height()) == (11, 6)
        _ORACLE_1024[t] = {"lbvh": ref, "hybrid": {"occupied": occ, "cell_size": 16,
                                                   "tree": shallow}}


@pytest.mark.parametrize("kind", ["lbvh", "hybrid"])
def test_config3_1080p_frame_vs_oracle(vs, vol1024, kind):
    u8, host = vol1024
    t = 0.3
    if t not in _ORACLE_1024:
        pytest.skip("needs test_config3_1024_indices_vs_oracle[0.3] in the same session")
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(t)
    idx = vs.build_index(kind, vs.classify(v, tf, dilate=True))
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
    rgba, samples = vs.render_float(v, tf, idx, cam)
    orgba, osamples = O.render(kind, host, tf.lut, _ORACLE_1024[t][kind], cam)
    np.testing.assert_array_equal(samples, osamples)
    np.testing.assert_array_equal(rgba, orgba)
    want = {"lbvh": 275332432, "hybrid": 773714751}[kind]  # SURVEY App. B frame samples
    assert int(samples.sum()) == want


@pytest.mark.parametrize("t", [0.3, 0.0])
def test_config3_1080p_early_ray_termination_vs_oracle(vs, vol1024, t):
    """Opt-in ERT (bench "ert" key, eps 5e-4) against the oracle's float RGBA at the north
    star's tolerance: every channel within 1e-3 (and within eps) of the reference integral, never
    more samples than the reference counts, on a 64-row band of the 1080p LBVH frame."""
    from paper_1912_09596_b200.render import RenderTarget, render_rows

    u8, host = vol1024
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction.ramp(t)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
    r0, r1 = 480, 544
    eps = 5e-4
    tgt = RenderTarget(1920, 1080, want_rgba64=True, want_samples=True)
    render_rows(v, tf, idx, cam, tgt, ert_eps=eps)
    rgba = tgt.rgba64.cpu().numpy().reshape(1080, 1920, 4)[r0:r1]
    samples = tgt.samples.cpu().numpy().reshape(1080, 1920)[r0:r1]
    ref = _oracle_lbvh(O.classify(host, tf.lut, dilate=True)[0])
    orgba, osamples = O.render("lbvh", host, tf.lut, ref, cam, rows=(r0, r1))
    err = float(np.max(np.abs(rgba - orgba.reshape(rgba.shape))))
    assert err <= eps <= 1e-3, err
    assert np.all(samples <= osamples.reshape(samples.shape))
    if t == 0.0:  # dense: saturating rays stop early (about a quarter fewer samples)
        assert int(samples.sum()) < 0.9 * int(osamples.sum())


# -- configs[4] ---------------------------------------------------------------------------------

def test_config4_four_channel_1024_row_band_vs_oracle(vs, vol1024):
    import sys
    from pathlib import Path

    from paper_1912_09596_b200.multichannel import classify_multi, render_float_multi
    from paper_1912_09596_b200.render import RowsDesc

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench as B

    chans = [vol1024] + [_blobs(1024, 25600, seed=7 + c) for c in range(1, 4)]
    vols = [vs.Volume.from_u8(u) for u, _ in chans]
    tfs = B.channel_tfs(4)[21]  # t = 0.4, the bench's sweep TFs
    idx = vs.build_index("lbvh", classify_multi(vols, tfs, dilate=True))
    # union classification: OR of the channels' visibility, then the 26-dilation
    union = np.zeros(vols[0].dims, bool)
    for (_, host), tf in zip(chans, tfs):
        union |= O.classify(host, tf.lut, dilate=False)[0]
    opaque = np.zeros((256, 4), np.float32)
    opaque[1:, 3] = 1.0
    bits, _ = O.classify(union.view(np.uint8), opaque, dilate=True)
    ref = _oracle_lbvh(bits)
    _same(idx, ref, LBVH, "4ch lbvh")
    cam = B.cameras(vols[0].dims)[21]
    band = 32  # image rows 512..543 (stripe 32, part 16)
    rows = RowsDesc(band, band, -(-cam.height // band), 16)
    rgba, samples = render_float_multi(vols, tfs, idx, cam, rows=rows)
    orgba, osamples = O.render_multi("lbvh", [h for _, h in chans], [tf.lut for tf in tfs], ref,
                                     cam, rows=(512, 512 + band))
    np.testing.assert_array_equal(samples, osamples)
    np.testing.assert_array_equal(rgba, orgba)
    assert int(samples.sum()) > 0


def test_lbvh_1024_device_properties(vs, vol1024):
    """Size-independent properties on the rebuild engine's own arrays (the graph-captured
    path the bench times): leaves in strictly increasing Morton order, internal boxes are the
    unions of their children."""
    import torch

    from paper_1912_09596_b200.engine import LbvhRebuilder
    from paper_1912_09596_b200.lbvh import morton_encode

    u8, _ = vol1024
    v = vs.Volume.from_u8(u8)
    rb = LbvhRebuilder(v)
    rb.rebuild(vs.TransferFunction.ramp(0.3).params())
    idx = rb.lbvh()
    n = idx.n_bricks
    assert n == 243434 and idx.node_count == 486867 and idx.height() == 22
    bc = idx.dev["brick_coords"][:n].long()
    codes = torch.from_numpy(morton_encode(*bc.cpu().numpy().T).astype(np.int64)).to(bc.device)
    assert bool((codes[1:] > codes[:-1]).all())
    lo, hi = idx.dev["lo"][:2 * n - 1], idx.dev["hi"][:2 * n - 1]
    left, right = idx.dev["left"][:n - 1].long(), idx.dev["right"][:n - 1].long()
    assert bool((lo[:n - 1] == torch.minimum(lo[left], lo[right])).all())
    assert bool((hi[:n - 1] == torch.maximum(hi[left], hi[right])).all())


def test_lbvh_1024_warm_rebuild_equals_cold(vs, vol1024):
    """The warm rebuild (per-volume presence masks, no volume read per TF) produces the cold
    rebuild's arrays and leaf-brick grid at every sweep TF, including non-monotone band TFs
    (where a per-brick min/max range test would not be exact)."""
    import torch

    from paper_1912_09596_b200.engine import LbvhRebuilder

    u8, _ = vol1024
    v = vs.Volume.from_u8(u8)
    cold, warm = LbvhRebuilder(v), LbvhRebuilder(v, warm=True)
    tfs = [vs.TransferFunction.ramp(t) for t in (0.6, 0.45, 0.3, 0.1, 0.0)]
    for lo_b, hi_b in ((180, 181), (90, 120), (3, 4)):
        lut = np.zeros((256, 4), np.float32)
        lut[lo_b:hi_b + 1] = 0.5
        tfs.append(vs.TransferFunction(lut))
    for tf in tfs:
        cold.rebuild(tf.params())
        warm.rebuild(tf.params())
        torch.cuda.synchronize()
        assert torch.equal(cold.info[:1], warm.info[:1])
        n = int(cold.info[0])
        m = max(2 * n - 1, 0)
        for f in LBVH:
            rows = n if f == "brick_coords" else m
            assert torch.equal(cold.tree[f][:rows], warm.tree[f][:rows]), f
        assert torch.equal(cold.brick_bits, warm.brick_bits)
    # multi-channel union (configs[4] semantics): warm == cold
    ch = [v, vs.Volume.from_u8(torch.flip(u8, dims=[0]).contiguous())]
    cold2, warm2 = LbvhRebuilder(ch), LbvhRebuilder(ch, warm=True)
    p = torch.cat([vs.TransferFunction.ramp(0.3).params(), vs.TransferFunction.ramp(0.5).params()])
    cold2.rebuild(p)
    warm2.rebuild(p)
    torch.cuda.synchronize()
    n = int(cold2.info[0])
    assert n > 0 and torch.equal(cold2.info[:1], warm2.info[:1])
    for f in LBVH:
        rows = n if f == "brick_coords" else 2 * n - 1
        assert torch.equal(cold2.tree[f][:rows], warm2.tree[f][:rows]), f
