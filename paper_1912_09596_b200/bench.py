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
