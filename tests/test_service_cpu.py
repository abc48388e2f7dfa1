"""Session-protocol host logic that needs no GPU: set_tf coalescing (service.py:171-187)."""

import json

from paper_1912_09596_b200.service import _coalesce


def test_coalesce_keeps_last_tf_of_each_run():
    tf = lambda k: json.dumps({"type": "set_tf", "rgba": k})  # noqa: E731
    cam = json.dumps({"type": "set_camera", "azimuth_deg": 1, "elevation_deg": 0, "zoom": 1})
    batch = [tf(1), tf(2), cam, tf(3), "not json", tf(4), tf(5)]
    assert _coalesce(batch) == [tf(2), cam, tf(3), "not json", tf(5)]
    assert _coalesce([]) == []
