"""Index-kind dispatch: the operator boundary of the hot path.

Drop-in for the dispatch half of voxelskip.bench (/root/reference/pkg/src/voxelskip/bench.py
:44-60, 161-183): ``INDEX_KINDS``, ``build_index(kind, b)`` and ``report_stats(index)`` with the
same kinds, defaults and errors; each builder runs on the GPU.
"""

from __future__ import annotations

import csv as _csv
import io as _io
import logging as _logging
import statistics as _statistics
import time as _time
from dataclasses import dataclass
from pathlib import Path

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


_log = _logging.getLogger(__name__)


# -- benchmark harness + CSV ------------------------------------------------
#
# The contract (bench.py:1-11, 42, 63-117 of the reference): one CSV row per index kind with
# the columns of CSV_HEADER, occupancy in percent of voxels visible under the undilated
# classification, build seconds as the median over ``reps`` builds, fps over a ``frames``-view
# orbit (azimuth 360 i / frames, elevation 0) at ``viewport`` square pixels.  Datasets are a
# raw file or a generator spec, TFs a JSON LUT or a preset.  Written here from that contract;
# the GPU build time includes the fused device classification the build consumes (a lazy
# BinaryVolume is evaluated inside the build), and every time is device-synchronised.

CSV_HEADER = "dataset,index,occupancy_pct,build_s,fps,nodes,height,samples"
_CSV_FORMATS = (str, str, "{:.4f}".format, "{:.6f}".format, "{:.4f}".format, str, str, str)


@dataclass
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
        for field, least in (("frames", 1), ("viewport", 16), ("reps", 1)):
            if getattr(self, field) < least:
                raise ValueError(f"{field} must be >= {least}")
        unknown = [k for k in self.kinds if k not in INDEX_KINDS]
        if unknown:
            raise ValueError(f"unknown index kind: {unknown[0]!r}")


@dataclass
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
        values = (self.dataset, self.index, self.occupancy_pct, self.build_s, self.fps,
                  self.nodes, self.height, self.samples)
        return [fmt(v) for fmt, v in zip(_CSV_FORMATS, values)]


def parse_dims(text: str):
    """``"64"`` -> (64, 64, 64); ``"8x9x10"`` -> (8, 9, 10)."""
    dims = [int(p) for p in text.lower().split("x")]
    if len(dims) not in (1, 3):
        raise ValueError(f"bad dims spec: {text!r}")
    return tuple(dims * 3 if len(dims) == 1 else dims)


def _generator_args(text: str) -> dict:
    args = {}
    for item in filter(None, text.split(",")):
        if "=" not in item:
            raise ValueError(f"bad generator argument: {item!r}")
        key, value = item.split("=", 1)
        args[key.strip()] = value.strip()
    return args


def _gen_menger(a):
    from .volume import gen_menger

    return gen_menger(int(a.get("level", 3)))


def _gen_shell(a):
    from .volume import gen_shell

    dims = parse_dims(a.get("dims", "128"))
    radius = float(a["radius"]) if "radius" in a else 0.375 * min(dims)
    return gen_shell(dims, radius=radius, thickness=float(a.get("thickness", 1)))


def _gen_blobs(a):
    from .volume import gen_blobs

    return gen_blobs(parse_dims(a.get("dims", "128")), n=int(a.get("n", 100)),
                     seed=int(a.get("seed", 0)))


_GENERATORS = {"menger": _gen_menger, "shell": _gen_shell, "blobs": _gen_blobs}


def load_dataset(spec: str):
    """A raw volume path, or ``[gen:]name[:key=value,...]`` with name menger (level=3),
    shell (dims=128, radius=0.375*min(dims), thickness=1) or blobs (dims=128, n=100, seed=0)."""
    from .volume import load_raw

    body = spec.removeprefix("gen:")
    name, _, args = body.partition(":")
    gen = _GENERATORS.get(name)
    return load_raw(spec) if gen is None else gen(_generator_args(args))


def load_tf(spec: str | None):
    """None / "ramp" -> the default ramp, "opaque" -> the opaque preset, else a LUT JSON file."""
    from .volume import TransferFunction

    presets = {None: TransferFunction.ramp, "ramp": TransferFunction.ramp,
               "opaque": TransferFunction.opaque}
    make = presets.get(spec)
    return make() if make is not None else TransferFunction.from_json(spec)


def _device_seconds(fn):
    import torch

    torch.cuda.synchronize()
    t0 = _time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, _time.perf_counter() - t0


def _median_build(kind, v, tf, reps):
    """Median wall time of ``reps`` TF-to-index builds; each rep classifies afresh (lazy
    classification: the build is where the device reads the volume)."""
    from .volume import classify

    def once():
        idx = build_index(kind, classify(v, tf, dilate=True))
        report_stats(idx)  # node counts/heights live on the device until read
        return idx

    runs = [_device_seconds(once) for _ in range(reps)]
    return runs[-1][0], _statistics.median(t for _, t in runs)


def _orbit(v, tf, index, cfg):
    """(frames/s, total samples) of the ``cfg.frames``-view orbit."""
    from .render import Camera, render_frame

    views = [Camera.orbit(v.dims, azimuth_deg=360.0 * i / cfg.frames, width=cfg.viewport)
             for i in range(cfg.frames)]
    samples, seconds = _device_seconds(
        lambda: sum(render_frame(v, tf, index, c, dt=cfg.dt).sample_count for c in views))
    return (cfg.frames / seconds if seconds > 0 else float("inf")), samples


def run_benchmark(cfg: BenchConfig) -> list:
    """One BenchRecord per kind of ``cfg.kinds``; the CSV goes to ``cfg.output`` if set."""
    from .volume import classify

    v, tf = load_dataset(cfg.dataset), load_tf(cfg.tf)
    nx, ny, nz = v.dims
    visible, classify_s = _device_seconds(
        lambda: classify(v, tf, dilate=False).base_count())
    occupancy_pct = 100.0 * visible / (nx * ny * nz)
    _log.info("classification: %.4f s, occupancy %.4f%%", classify_s, occupancy_pct)
    records = []
    for kind in cfg.kinds:
        index, build_s = _median_build(kind, v, tf, cfg.reps)
        fps, samples = _orbit(v, tf, index, cfg)
        st = report_stats(index)
        _log.info("%s: build %.6f s, %.2f fps, %d samples", kind, build_s, fps, samples)
        records.append(BenchRecord(cfg.dataset, kind, occupancy_pct, build_s, fps,
                                   st["node_count"], st["height"], samples))
    if cfg.output is not None:
        Path(cfg.output).write_text(to_csv(records))
    return records


def to_csv(records) -> str:
    out = _io.StringIO()
    w = _csv.writer(out, lineterminator="\n")
    w.writerow(CSV_HEADER.split(","))
    w.writerows(r.csv_row() for r in records)
    return out.getvalue()
