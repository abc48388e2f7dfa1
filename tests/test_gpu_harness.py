"""Raw I/O, generators and the benchmark harness on the GPU path."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import unpack_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    return vs


def test_generators_match_reference_fixtures(vs, scenes):
    shell = vs.gen_shell((32, 32, 32), radius=12.0, thickness=2.0)
    np.testing.assert_array_equal(shell.bins.cpu().numpy(), scenes["shell_u8"])
    menger = vs.gen_menger(2)
    np.testing.assert_array_equal(menger.bins.cpu().numpy(), scenes["menger_u8"])
    m3 = vs.gen_menger(3)  # test_volume.py:248-251: occupancy exactly 8000/19683
    assert vs.occupancy(vs.classify(m3, vs.TransferFunction.opaque())) == 8000 / 19683


def test_blobs_u8_matches_reference(vs, blobs64):
    from paper_1912_09596_b200.synth import gen_blobs_u8

    u8 = gen_blobs_u8((64, 64, 64), 16, seed=7, sigma=3.0).cpu().numpy()
    assert (u8 == blobs64["u8"]).mean() > 0.999  # summation order may flip rare ties


def test_raw_round_trip(vs, tmp_path, blobs64):
    v = vs.Volume.from_u8(blobs64["u8"])
    vs.save_raw(v, tmp_path / "b.raw")
    meta = json.loads((tmp_path / "b.raw.json").read_text())
    assert meta == {"dims": [64, 64, 64], "bits": 8, "endian": "little"}
    disk = np.frombuffer((tmp_path / "b.raw").read_bytes(), np.uint8).reshape((64, 64, 64), order="F")
    np.testing.assert_array_equal(disk, blobs64["u8"])
    w = vs.load_raw(tmp_path / "b.raw")
    assert w.field is None
    np.testing.assert_array_equal(w.bins.cpu().numpy(), blobs64["u8"])
    # 16-bit: normalised in float64, narrowed to float32 (volume.py:193)
    rng = np.random.default_rng(3)
    u16 = rng.integers(0, 65536, size=(5, 6, 7)).astype("<u2")
    (tmp_path / "c.raw").write_bytes(u16.flatten(order="F").tobytes())
    c = vs.load_raw(tmp_path / "c.raw", {"dims": [5, 6, 7], "bits": 16})
    want = (u16.astype(np.float64) / 65535.0).astype(np.float32)
    np.testing.assert_array_equal(c.data, want)
    with pytest.raises(vs.VolumeFormatError):
        vs.load_raw(tmp_path / "c.raw", {"dims": [5, 6, 8], "bits": 16})
    with pytest.raises(vs.UnsupportedFormatError):
        vs.load_raw(tmp_path / "c.raw", {"dims": [5, 6, 7], "bits": 12})


def test_run_benchmark_csv(vs, tmp_path):
    out = tmp_path / "bench.csv"
    cfg = vs.BenchConfig("menger:level=3", tf="opaque", kinds=("naive", "grid", "lbvh", "hybrid"),
                         frames=4, viewport=32, reps=2, output=str(out))
    recs = vs.run_benchmark(cfg)
    assert [r.index for r in recs] == ["naive", "grid", "lbvh", "hybrid"]
    occ = 100.0 * 8000 / 19683
    assert all(abs(r.occupancy_pct - occ) < 1e-9 for r in recs)
    assert recs[0].nodes == 0 and recs[2].nodes > 0 and recs[3].height > 0
    # skipping never changes the image, so every kind takes at most naive's samples
    assert all(r.samples <= recs[0].samples for r in recs)
    assert out.read_text().splitlines()[0] == vs.CSV_HEADER
