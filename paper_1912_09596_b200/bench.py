"""Index-kind dispatch: the operator boundary of the hot path.

Drop-in for the dispatch half of voxelskip.bench (/root/reference/pkg/src/voxelskip/bench.py
:44-60, 161-183): ``INDEX_KINDS``, ``build_index(kind, b)`` and ``report_stats(index)`` with the
same kinds, defaults and errors; each builder runs on the GPU.
"""

from __future__ import annotations

from .lbvh import Lbvh, build_lbvh, flag_bricks
from .svt import MacroGrid, derive_macro_grid
from .volume import BinaryVolume

INDEX_KINDS = (
    "naive",
    "grid",
    "lbvh",
    "kd-shallow",
    "kd-deep-mls32",
    "kd-deep-mls128",
    "kd-binned-mls32",
    "hybrid",
)


def index_kind(index) -> str:
    """render.py:44-55."""
    if index is None:
        return "naive"
    if isinstance(index, MacroGrid):
        return "grid"
    if isinstance(index, Lbvh):
        return "lbvh"
    name = type(index).__name__
    if name == "KdTree":
        return "kd"
    if name == "HybridGrid":
        return "hybrid"
    raise TypeError(f"not a spatial index: {name}")


def build_index(kind: str, b: BinaryVolume):
    """One index of the requested kind over a classification (bench.py:161-173)."""
    if kind == "naive":
        return None
    if kind == "grid":
        return derive_macro_grid(b, 16)
    if kind == "lbvh":
        return build_lbvh(flag_bricks(b))
    if kind == "hybrid" or kind in ("kd-shallow", "kd-deep-mls32", "kd-deep-mls128",
                                    "kd-binned-mls32"):
        from . import kdtree  # noqa: F401  (SVT k-d builders)

        return kdtree.build_index_kind(kind, b)
    raise ValueError(f"unknown index kind: {kind!r}")


def report_stats(index) -> dict[str, int]:
    """Node count and height; 0/0 for indices without a tree (bench.py:176-183)."""
    kind = index_kind(index)
    if kind in ("naive", "grid"):
        return {"node_count": 0, "height": 0}
    tree = index.tree if kind == "hybrid" else index
    return {"node_count": tree.node_count, "height": tree.height()}


# -- benchmark harness + CSV (bench.py:42, 63-158, 186-249) ----------------

import csv as _csv
import io as _io
import logging as _logging
import statistics as _statistics
import time as _time
from dataclasses import dataclass as _dataclass

_log = _logging.getLogger(__name__)

CSV_HEADER = "dataset,index,occupancy_pct,build_s,fps,nodes,height,samples"


@_dataclass
class BenchConfig:
    dataset: str
    tf: str | None = None
    kinds: tuple = ("naive",)
    frames: int = 36
    viewport: int = 1024
    dt: float = 0.5
    reps: int = 3
    output: str | None = None

    def __post_init__(self):
        if self.frames < 1:
            raise ValueError("frames must be >= 1")
        if self.viewport < 16:
            raise ValueError("viewport must be >= 16")
        if self.reps < 1:
            raise ValueError("reps must be >= 1")
        for kind in self.kinds:
            if kind not in INDEX_KINDS:
                raise ValueError(f"unknown index kind: {kind!r}")


@_dataclass
class BenchRecord:
    dataset: str
    index: str
    occupancy_pct: float
    build_s: float
    fps: float
    nodes: int
    height: int
    samples: int

    def csv_row(self) -> list:
        return [self.dataset, self.index, f"{self.occupancy_pct:.4f}", f"{self.build_s:.6f}",
                f"{self.fps:.4f}", str(self.nodes), str(self.height), str(self.samples)]


def parse_dims(text: str):
    parts = text.lower().split("x")
    if len(parts) == 1:
        d = int(parts[0])
        return (d, d, d)
    if len(parts) == 3:
        return tuple(int(p) for p in parts)
    raise ValueError(f"bad dims spec: {text!r}")


def load_dataset(spec: str):
    """A raw volume file or a generator spec ``name:key=value,...`` (bench.py:120-148)."""
    from .volume import gen_blobs, gen_menger, gen_shell, load_raw

    text = spec[4:] if spec.startswith("gen:") else spec
    name, _, rest = text.partition(":")
    if name in ("menger", "shell", "blobs"):
        kv = {}
        if rest:
            for item in rest.split(","):
                key, sep, value = item.partition("=")
                if not sep:
                    raise ValueError(f"bad generator argument: {item!r}")
                kv[key.strip()] = value.strip()
        if name == "menger":
            return gen_menger(int(kv.get("level", "3")))
        if name == "shell":
            dims = parse_dims(kv.get("dims", "128"))
            radius = float(kv["radius"]) if "radius" in kv else 0.375 * min(dims)
            return gen_shell(dims, radius=radius, thickness=float(kv.get("thickness", "1")))
        return gen_blobs(parse_dims(kv.get("dims", "128")), n=int(kv.get("n", "100")),
                         seed=int(kv.get("seed", "0")))
    return load_raw(spec)


def load_tf(spec: str | None):
    """A LUT JSON file, a preset (``ramp``/``opaque``) or the default ramp (bench.py:151-158)."""
    from .volume import TransferFunction

    if spec is None or spec == "ramp":
        return TransferFunction.ramp()
    if spec == "opaque":
        return TransferFunction.opaque()
    return TransferFunction.from_json(spec)


def _sync():
    import torch

    torch.cuda.synchronize()


def run_benchmark(cfg: BenchConfig) -> list:
    """Classify once, then per kind: timed builds (median of reps, device-synchronised), a
    rotating render pass, one record; CSV when cfg.output is set (bench.py:186-240)."""
    from .render import Camera, render_frame
    from .volume import classify, occupancy

    v = load_dataset(cfg.dataset)
    tf = load_tf(cfg.tf)
    _sync()
    t0 = _time.perf_counter()
    occ_pct = 100.0 * occupancy(classify(v, tf, dilate=False))
    b = classify(v, tf, dilate=True)
    _sync()
    _log.info("classification (plain + dilated): %.4f s", _time.perf_counter() - t0)
    cameras = [Camera.orbit(v.dims, azimuth_deg=360.0 * i / cfg.frames, width=cfg.viewport)
               for i in range(cfg.frames)]
    records = []
    for kind in cfg.kinds:
        times, index = [], None
        for _ in range(cfg.reps):
            _sync()
            t0 = _time.perf_counter()
            index = build_index(kind, classify(v, tf, dilate=True) if kind != "naive" else b)
            report_stats(index)  # forces completion (node counts live on the device)
            _sync()
            times.append(_time.perf_counter() - t0)
        build_s = _statistics.median(times)
        stats = report_stats(index)
        samples = 0
        _sync()
        t0 = _time.perf_counter()
        for cam in cameras:
            samples += render_frame(v, tf, index, cam, dt=cfg.dt).sample_count
        render_s = _time.perf_counter() - t0
        fps = cfg.frames / render_s if render_s > 0 else float("inf")
        records.append(BenchRecord(dataset=cfg.dataset, index=kind, occupancy_pct=occ_pct,
                                   build_s=build_s, fps=fps, nodes=stats["node_count"],
                                   height=stats["height"], samples=samples))
    if cfg.output is not None:
        from pathlib import Path

        Path(cfg.output).write_text(to_csv(records))
    return records


def to_csv(records) -> str:
    buf = _io.StringIO()
    writer = _csv.writer(buf, lineterminator="\n")
    writer.writerow(CSV_HEADER.split(","))
    for rec in records:
        writer.writerow(rec.csv_row())
    return buf.getvalue()
