"""k-d trees over occupancy classifications on the B200, drop-in for voxelskip.kdtree
(/root/reference/pkg/src/voxelskip/kdtree.py).

KdTree keeps the reference's flat row layout (DFS preorder, row 0 = root): lo/hi (m,3) int32,
axis (m,) int8 (-1 = leaf), plane/left/right (m,) int32 (-1 = dropped child).  Device copies
feed the renderer; host arrays are materialised lazily.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .volume import Aabb

DEFAULT_CELL_SIZE = 8
DEFAULT_BINS = 4
MAX_NZ = 1024  # vs_kd_build / vs_kd_best_plane: a z row is at most one warp of 32-bit words


@dataclass(frozen=True)
class BuildParams:
    """Knobs for build_kdtree (kdtree.py:43-73)."""

    mode: str = "shallow"
    max_leaf_size: int | None = None
    builder: str = "sweep"
    bins: int = DEFAULT_BINS
    cell_size: int = DEFAULT_CELL_SIZE

    def __post_init__(self):
        if self.mode not in ("shallow", "deep"):
            raise ValueError(f"unknown mode: {self.mode!r}")
        if self.builder not in ("sweep", "binned"):
            raise ValueError(f"unknown builder: {self.builder!r}")
        if self.max_leaf_size is not None:
            if self.mode != "deep":
                raise ValueError("max_leaf_size only applies to deep trees")
            if self.max_leaf_size < 1:
                raise ValueError("max_leaf_size must be positive")
        if self.bins < 2:
            raise ValueError("bins must be >= 2")
        if self.cell_size < 1:
            raise ValueError("cell_size must be positive")


@dataclass(frozen=True)
class SplitPlane:
    """An axis-aligned cut: voxels with coordinate < position go left (kdtree.py:76-82)."""

    axis: int
    position: int
    cost: int


class KdTree:
    """Flat node arrays, row 0 the root unless empty (kdtree.py:85-127)."""

    _FIELDS = ("lo", "hi", "axis", "plane", "left", "right")

    def __init__(self, lo=None, hi=None, axis=None, plane=None, left=None, right=None,
                 root: int = -1, dims=(0, 0, 0), *, dev: dict | None = None,
                 height: int | None = None):
        self.root = int(root)
        self.dims = tuple(int(d) for d in dims)
        self._host = {}
        if dev is None:
            self._host = {
                "lo": np.asarray(lo, np.int32).reshape(-1, 3),
                "hi": np.asarray(hi, np.int32).reshape(-1, 3),
                "axis": np.asarray(axis, np.int8).reshape(-1),
                "plane": np.asarray(plane, np.int32).reshape(-1),
                "left": np.asarray(left, np.int32).reshape(-1),
                "right": np.asarray(right, np.int32).reshape(-1),
            }
            self._m = len(self._host["axis"])
        else:
            self._m = int(dev["axis"].shape[0])
        self._dev = dev
        self._height = height

    def __getattr__(self, name):
        if name in KdTree._FIELDS:
            h = self.__dict__["_host"]
            if name not in h:
                h[name] = self.__dict__["_dev"][name].cpu().numpy()
            return h[name]
        raise AttributeError(name)

    def device_arrays(self) -> dict:
        if self._dev is None:
            dev = _lib.device()
            self._dev = {k: torch.from_numpy(np.ascontiguousarray(self._host[k])).to(dev)
                         for k in KdTree._FIELDS}
        return self._dev

    @property
    def node_count(self) -> int:
        return self._m

    def is_leaf(self, i: int) -> bool:
        return bool(self.axis[i] < 0)

    def node_box(self, i: int) -> Aabb:
        return Aabb(tuple(int(v) for v in self.lo[i]), tuple(int(v) for v in self.hi[i]))

    def leaf_mask(self) -> np.ndarray:
        return self.axis < 0

    def height(self) -> int:
        """Nodes on the longest root-to-leaf path (kdtree.py:115-127)."""
        if self._height is None:
            if self.node_count == 0:
                self._height = 0
            else:
                left, right = self.left, self.right
                best, stack = 0, [(self.root, 1)]
                while stack:
                    i, d = stack.pop()
                    best = max(best, d)
                    for c in (int(left[i]), int(right[i])):
                        if c >= 0:
                            stack.append((c, d + 1))
                self._height = best
        return self._height


def empty_kdtree(dims) -> KdTree:
    z3 = np.zeros((0, 3), np.int32)
    z = np.zeros(0, np.int32)
    return KdTree(z3, z3, np.zeros(0, np.int8), z, z, z, -1, dims)


def build_kdtree(g, params: BuildParams | None = None) -> KdTree:
    """Top-down build over a table grid (kdtree.py:387-498) on the device: level-synchronous
    split search (vs_kd_build), rows in the reference's DFS preorder."""
    import ctypes as C

    from ._lib import call, ptr, query, stream

    params = params or BuildParams()
    b = g.binary
    nx, ny, nz = g.dims
    if nz > MAX_NZ:
        # the span passes give one z row to one warp (32 lanes x 32-bit words)
        raise ValueError(f"build_kdtree supports nz <= {MAX_NZ} (got dims {g.dims}); "
                         "store the longest axis first (x or y)")
    h = C.c_void_p()
    try:
        packed = b.packed()
        call("vs_kd_build_bbox", ptr(packed), nx, ny, nz,
             ptr(b._bbox) if getattr(b, "_bbox", None) is not None else None,
             int(params.mode == "deep"),
             -1 if params.max_leaf_size is None else int(params.max_leaf_size),
             int(params.builder == "binned"), int(params.bins), int(params.cell_size),
             C.byref(h), stream())
        m, root, height = C.c_int64(), C.c_int(), C.c_int()
        call("vs_kd_result_info", h, C.byref(m), C.byref(root), C.byref(height))
        m = int(m.value)
        if m == 0:
            return empty_kdtree(g.dims)
        dev = _lib.device()
        d = {"lo": torch.empty((m, 3), dtype=torch.int32, device=dev),
             "hi": torch.empty((m, 3), dtype=torch.int32, device=dev),
             "axis": torch.empty(m, dtype=torch.int8, device=dev),
             "plane": torch.empty(m, dtype=torch.int32, device=dev),
             "left": torch.empty(m, dtype=torch.int32, device=dev),
             "right": torch.empty(m, dtype=torch.int32, device=dev)}
        call("vs_kd_result_copy", h, ptr(d["lo"]), ptr(d["hi"]), ptr(d["axis"]), ptr(d["plane"]),
             ptr(d["left"]), ptr(d["right"]), stream())
        torch.cuda.current_stream().synchronize()
    finally:
        if h.value:
            _lib.lib().vs_kd_result_free(h)
    return KdTree(root=int(root.value), dims=g.dims, dev=d, height=int(height.value))


_KD_PARAMS = {
    "kd-shallow": BuildParams(mode="shallow"),
    "kd-deep-mls32": BuildParams(mode="deep", max_leaf_size=32),
    "kd-deep-mls128": BuildParams(mode="deep", max_leaf_size=128),
    "kd-binned-mls32": BuildParams(mode="deep", max_leaf_size=32, builder="binned"),
}


def build_index_kind(kind: str, b):
    """bench.py:166-172 for the table-based kinds."""
    from .hybrid import build_hybrid
    from .svt import build_svt_grid

    if kind == "hybrid":
        return build_hybrid(build_svt_grid(b), b)
    return build_kdtree(build_svt_grid(b), _KD_PARAMS[kind])


@dataclass
class CellBoxList:
    """Tight flag bounds of every coarse cell, sorted by cell Morton code (kdtree.py:268-282).
    Rows for unoccupied cells are placeholders; consult ``occupied`` first."""

    cell_size: int
    cells_dims: tuple
    dims: tuple
    codes: np.ndarray
    coords: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    occupied: np.ndarray
    binary: object = None  # the classification the boxes came from (device bits)


def precompute_cell_boxes(b, cell_size: int = DEFAULT_CELL_SIZE) -> CellBoxList:
    """Per-cell tight boxes in one device pass (vs_cell_boxes), rows in Morton order."""
    from ._lib import call, ptr, stream
    from .lbvh import morton_encode

    cs = int(cell_size)
    dims = b.dims
    nc = tuple(-(-d // cs) for d in dims)
    n = nc[0] * nc[1] * nc[2]
    dev = _lib.device()
    lo = torch.empty((n, 3), dtype=torch.int32, device=dev)
    hi = torch.empty((n, 3), dtype=torch.int32, device=dev)
    occ = torch.empty(n, dtype=torch.uint8, device=dev)
    call("vs_cell_boxes", ptr(b.packed()), *dims, cs, ptr(lo), ptr(hi), ptr(occ), stream())
    cx, cy, cz = np.indices(nc)
    coords = np.stack([cx, cy, cz], axis=-1).reshape(-1, 3)
    codes = np.asarray(morton_encode(coords[:, 0], coords[:, 1], coords[:, 2]), np.uint32)
    order = np.argsort(codes, kind="stable")
    return CellBoxList(cell_size=cs, cells_dims=nc, dims=dims, codes=codes[order],
                       coords=coords[order].astype(np.int32), lo=lo.cpu().numpy()[order],
                       hi=hi.cpu().numpy()[order], occupied=occ.cpu().numpy().view(bool)[order],
                       binary=b)


def _best_plane(b, box, binned: int, bins: int, cs: int):
    import ctypes as C

    from ._lib import call, ptr, stream

    bx = (C.c_int * 6)(*[int(v) for v in list(box.lo) + list(box.hi)])
    out = (C.c_longlong * 4)()
    nx, ny, nz = b.dims
    call("vs_kd_best_plane", ptr(b.packed()), nx, ny, nz, C.addressof(bx), int(binned),
         int(bins), int(cs), C.addressof(out), stream())
    if not out[0]:
        return None
    return SplitPlane(axis=int(out[1]), position=int(out[2]), cost=int(out[3]))


def sweep_best_plane(g, box) -> SplitPlane | None:
    """Exhaustive search for the cut minimising vol(tight left) + vol(tight right); None when
    no cut strictly beats the box's own tight volume; ties to the lower axis then position
    (kdtree.py:244-262)."""
    return _best_plane(g.binary, box, 0, DEFAULT_BINS, DEFAULT_CELL_SIZE)


def binned_best_plane(cells: CellBoxList, box, bins: int = DEFAULT_BINS) -> SplitPlane | None:
    """bins-1 snapped candidate cuts per axis with child bounds from the per-cell boxes
    (kdtree.py:371-381)."""
    if cells.binary is None:
        raise ValueError("CellBoxList was not built by precompute_cell_boxes")
    return _best_plane(cells.binary, box, 1, bins, cells.cell_size)


# -- host helpers the reference exposes at module level (its tests import them) -------------

def _snapped_positions(lo: int, hi: int, bins: int, cell_size: int) -> list[int]:
    """Candidate cuts of the binned search (kdtree.py:346-350): the bins-1 equal divisions of
    [lo, hi) rounded half-up to the cell lattice in IEEE double, strictly inside the box,
    deduplicated and ascending.  The device evaluates the same expression (k_decide_binned)."""
    import math

    step = (hi - lo) / bins
    cuts = set()
    for j in range(1, bins):
        p = int(math.floor((lo + j * step) / cell_size + 0.5)) * cell_size
        if lo < p < hi:
            cuts.add(p)
    return sorted(cuts)


def _cells_reduce(cells: CellBoxList, region: Aabb) -> Aabb | None:
    """Bounds of ``region`` from the per-cell tight boxes (kdtree.py:323-343): the union of the
    occupied cells whose lattice footprint meets the region, clipped back to the region; None
    when nothing remains.  Host mirror of the device's cell-slab reduction."""
    cs = cells.cell_size
    first = np.array([max(v // cs, 0) for v in region.lo])
    last = np.array([min((v - 1) // cs, n - 1) for v, n in zip(region.hi, cells.cells_dims)])
    if np.any(first > last):
        return None
    inside = cells.occupied & np.all((cells.coords >= first) & (cells.coords <= last), axis=1)
    if not inside.any():
        return None
    lo = np.maximum(cells.lo[inside].min(axis=0), region.lo)
    hi = np.minimum(cells.hi[inside].max(axis=0), region.hi)
    if np.any(lo >= hi):
        return None
    return Aabb(tuple(int(v) for v in lo), tuple(int(v) for v in hi))
