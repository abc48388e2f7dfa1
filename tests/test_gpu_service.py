"""The interactive session on the GPU path: protocol behaviour of service.py:128-168 and frame
equality with an offline render (test_service.py:146-155 in the reference)."""

from __future__ import annotations

import json
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_09596_b200 as vs

    return vs


def test_session_protocol(vs, blobs64):
    from paper_1912_09596_b200.service import Session, handle_message

    v = vs.Volume.from_u8(blobs64["u8"])
    s = Session(v, kind="lbvh", viewport=48)
    assert handle_message(s, '{"type": "ping"}')[0].payload == {"type": "pong"}
    assert handle_message(s, "{bad")[0].payload["type"] == "error"
    assert handle_message(s, '[1, 2]')[0].payload["type"] == "error"
    assert handle_message(s, '{"type": "nope"}')[0].payload["type"] == "error"
    bad = handle_message(s, json.dumps({"type": "set_tf", "rgba": [[0, 0, 0, 2]] * 256}))
    assert bad[0].payload["type"] == "error"
    lut = blobs64["ramp03_lut"]
    replies = handle_message(s, json.dumps({"type": "set_tf", "rgba": lut.tolist()}))
    stats, frame = replies[0].payload, replies[1].payload
    assert stats["type"] == "stats"
    assert stats["occupancy_pct"] == pytest.approx(100.0 * float(blobs64["ramp03_occupancy"]))
    ref_idx = vs.build_index("lbvh", vs.classify(v, vs.TransferFunction(lut), dilate=True))
    assert stats["nodes"] == ref_idx.node_count and stats["height"] == ref_idx.height()
    assert frame[:4] == b"FRME"
    w, h, seq = struct.unpack("<III", frame[4:16])
    assert (w, h) == (48, 48) and seq == 1
    # the served frame against the CPU oracle (not against the package's own render_frame)
    from oracle import oracle as O

    obits, _ = O.classify(blobs64["u8"], lut, dilate=True)
    coords, codes = O.flag_bricks(obits, 8)
    otree = O.build_lbvh(coords, codes, 8, v.dims)
    assert stats["nodes"] == otree["node_count"] and stats["height"] == otree["height"]
    cam = vs.Camera.orbit(v.dims, 0.0, 0.0, 1.0, width=48)
    orgba, osamples = O.render("lbvh", blobs64["u8"], lut, otree, cam, nthreads=4)
    np.testing.assert_array_equal(np.frombuffer(frame[16:], np.uint8).reshape(48, 48, 4),
                                  O.quantize_rgba(orgba))
    assert stats["samples"] == int(osamples.sum())
    _, plain_count = O.classify(blobs64["u8"], lut, dilate=False)
    assert stats["occupancy_pct"] == pytest.approx(100.0 * plain_count / 64 ** 3, rel=1e-12)
    r = handle_message(s, {"type": "set_camera", "azimuth_deg": 30, "elevation_deg": 10, "zoom": 1.5})
    assert r[0].kind == "binary" and struct.unpack("<III", r[0].payload[4:16])[2] == 2
    assert handle_message(s, {"type": "set_camera", "azimuth_deg": 0, "elevation_deg": 0,
                              "zoom": 0})[0].payload["type"] == "error"
    r = handle_message(s, {"type": "set_index", "kind": "kd-deep-mls32"})
    assert r[0].payload["type"] == "stats" and r[0].payload["classify_ms"] == 0.0
    okd = O.kd_build(obits, mode="deep", max_leaf_size=32)
    assert r[0].payload["nodes"] == okd["node_count"] and r[0].payload["height"] == okd["height"]
    cam = vs.Camera.orbit(v.dims, 30.0, 10.0, 1.5, width=48)
    orgba, osamples = O.render("kd", blobs64["u8"], lut, okd, cam, nthreads=4)
    np.testing.assert_array_equal(np.frombuffer(r[1].payload[16:], np.uint8).reshape(48, 48, 4),
                                  O.quantize_rgba(orgba))
    assert struct.unpack("<III", r[1].payload[4:16])[2] == 3
    assert handle_message(s, {"type": "set_index", "kind": "octree"})[0].payload["type"] == "error"
    assert handle_message(s, {"type": "set_tf"})[0].payload["type"] == "error"  # missing rgba
    assert handle_message(s, {"type": "set_camera", "azimuth_deg": float("nan"),
                              "elevation_deg": 0, "zoom": 1})[0].payload["type"] == "error"
