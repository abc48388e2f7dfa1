"""Benchmark-harness host logic (bench.py:63-158, 243-249 in the reference), no GPU needed."""

import pytest

from paper_1912_09596_b200.bench import (CSV_HEADER, BenchConfig, BenchRecord, load_tf,
                                         parse_dims, to_csv)


def test_config_validation():
    with pytest.raises(ValueError):
        BenchConfig("menger:level=2", frames=0)
    with pytest.raises(ValueError):
        BenchConfig("menger:level=2", viewport=8)
    with pytest.raises(ValueError):
        BenchConfig("menger:level=2", reps=0)
    with pytest.raises(ValueError):
        BenchConfig("menger:level=2", kinds=("octree",))
    BenchConfig("menger:level=2", kinds=("naive", "lbvh", "hybrid"))


def test_csv_and_dims():
    rec = BenchRecord("menger:level=2", "lbvh", 12.345678, 0.0012345678, 99.99999, 7, 3, 123)
    text = to_csv([rec])
    lines = text.splitlines()
    assert lines[0] == CSV_HEADER
    assert lines[1] == "menger:level=2,lbvh,12.3457,0.001235,100.0000,7,3,123"
    assert parse_dims("64") == (64, 64, 64) and parse_dims("8x9x10") == (8, 9, 10)
    with pytest.raises(ValueError):
        parse_dims("8x9")


def test_load_tf_presets(tmp_path):
    assert load_tf(None).lut[200, 3] > 0 and load_tf("opaque").lut[0, 3] == 0
    p = tmp_path / "tf.json"
    load_tf("ramp").to_json(p)
    assert (load_tf(str(p)).lut == load_tf("ramp").lut).all()
