"""Brick LBVH on the B200: flag, Morton-order, Karras radix tree, refit.

Drop-in for voxelskip.lbvh (/root/reference/pkg/src/voxelskip/lbvh.py): same names, array
layouts and exceptions.  Device pipeline (csrc/classify.cu, csrc/lbvh.cu):

  flag_bricks(b, 8) on a lazy classification -> vs_classify_summary (one pass over the u8
      volume) -> vs_summary_to_bitmap (dilated brick vote into a Morton-addressed bitmap)
  flag_bricks(b, bs) otherwise -> vs_vote_cells over packed bits -> vs_flags_to_bitmap
  build_lbvh(bricks) -> vs_lbvh_from_bitmap (rank = sorted order, leaves, Karras, refit) or,
      for a BrickSet built by hand, vs_lbvh_from_bricks (CUB radix sort of code<<32|index).

Results stay on the device; host numpy arrays are produced on first attribute access.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, stream
from .volume import Aabb, BinaryVolume

DEFAULT_BRICK_SIZE = 8
MORTON_AXIS_BITS = 10


class MortonRangeError(ValueError):
    """Coordinate outside the 10-bit-per-axis Morton budget."""


def _spread_bits(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x3FF)
    for shift, mask in ((16, 0x030000FF), (8, 0x0300F00F), (4, 0x030C30C3), (2, 0x09249249)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def _compact_bits(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0x09249249)
    for shift, mask in ((2, 0x030C30C3), (4, 0x0300F00F), (8, 0x030000FF), (16, 0x3FF)):
        v = (v | (v >> np.uint64(shift))) & np.uint64(mask)
    return v


def morton_encode(x, y, z):
    """x -> code bit 3i, y -> 3i+1, z -> 3i+2 (lbvh.py:44-55); scalars or arrays."""
    xa, ya, za = (np.asarray(c, dtype=np.int64) for c in (x, y, z))
    for c in (xa, ya, za):
        if c.size and (c.min() < 0 or c.max() >= 1 << MORTON_AXIS_BITS):
            raise MortonRangeError("coordinates must be in [0, 1024)")
    code = (_spread_bits(xa) | (_spread_bits(ya) << np.uint64(1)) |
            (_spread_bits(za) << np.uint64(2))).astype(np.uint32)
    return int(code) if code.ndim == 0 else code


def morton_decode(code):
    """Inverse of morton_encode (lbvh.py:58-66)."""
    c = np.asarray(code, dtype=np.uint64)
    x, y, z = (_compact_bits(c >> np.uint64(k)) for k in range(3))
    if c.ndim == 0:
        return int(x), int(y), int(z)
    return x.astype(np.int64), y.astype(np.int64), z.astype(np.int64)


class BrickSet:
    """The non-empty bricks of a classification with their Morton codes (lbvh.py:69-80).

    ``coords`` (n,3) int32 in scan (C) order and ``codes`` (n,) uint32.  Bricks produced by
    flag_bricks also carry the device Morton bitmap that build_lbvh consumes directly."""

    def __init__(self, brick_size: int, dims, coords=None, codes=None, *, _bitmap=None):
        self.brick_size = int(brick_size)
        self.dims = tuple(int(d) for d in dims)
        self._bitmap = _bitmap  # (bitmap, tile_counts, P, nb) or None
        self._coords = None if coords is None else np.asarray(coords, dtype=np.int32).reshape(-1, 3)
        self._codes = None if codes is None else np.asarray(codes, dtype=np.uint32).reshape(-1)
        self._n = None if self._coords is None else len(self._coords)
        if self._coords is not None and self._codes is not None and \
                len(self._coords) != len(self._codes):
            raise ValueError("coords and codes must have the same length")

    def _materialise(self):
        bitmap, tiles, P, nb = self._bitmap
        dev = bitmap.device
        ncell = nb[0] * nb[1] * nb[2]
        coords = torch.empty((ncell, 3), dtype=torch.int32, device=dev)
        codes = torch.empty(ncell, dtype=torch.int32, device=dev)
        n_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb = query("vs_bricks_workspace", *nb)
        ws = _lib.workspace(wsb)
        call("vs_bricks_from_bitmap", ptr(bitmap), *nb, P, ptr(coords), ptr(codes), ptr(n_dev),
             ptr(ws), wsb, stream())
        n = int(n_dev.item())
        self._coords = coords[:n].cpu().numpy()
        self._codes = codes[:n].cpu().numpy().view(np.uint32)
        self._n = n

    @property
    def coords(self) -> np.ndarray:
        if self._coords is None:
            self._materialise()
        return self._coords

    @property
    def codes(self) -> np.ndarray:
        if self._codes is None:
            self._materialise()
        return self._codes

    @property
    def count(self) -> int:
        if self._n is None:
            if self._bitmap is not None:
                self._n = int(self._bitmap[1].sum().item())
            else:
                self._n = len(self.coords)
        return self._n


def _brick_grid(dims, bs):
    nb = tuple(-(-d // bs) for d in dims)
    if max(nb) > 1 << MORTON_AXIS_BITS:
        raise MortonRangeError(f"brick grid {nb} exceeds 1024 per axis")
    return nb


def flag_bricks(b: BinaryVolume, brick_size: int = DEFAULT_BRICK_SIZE) -> BrickSet:
    """Vote per brick (OR over its flags) and compact to the non-empty ones, in scan order
    (lbvh.py:83-102)."""
    if brick_size < 1:
        raise ValueError("brick_size must be >= 1")
    bs = int(brick_size)
    dims = b.dims
    nb = _brick_grid(dims, bs)
    P = query("vs_morton_side", *nb)
    dev = _lib.device()
    bitmap = torch.empty(P * P * P // 32, dtype=torch.int32, device=dev)
    tiles = torch.empty(P * P * P // 512, dtype=torch.int32, device=dev)
    nx, ny, nz = dims
    grid = None
    if bs == 8 and b.lazy and b.summary_ok():
        words = (nb[0] * nb[1] * nb[2] + 31) // 32
        grid = torch.empty(max(words, 1), dtype=torch.int32, device=dev)
        b.vote_bitmap(P, bitmap, tiles, grid=grid)
    else:
        flags = torch.empty(nb, dtype=torch.uint8, device=dev)
        call("vs_vote_cells", ptr(b.packed()), nx, ny, nz, bs, ptr(flags), stream())
        call("vs_flags_to_bitmap", ptr(flags), *nb, P, ptr(bitmap), ptr(tiles), stream())
    out = BrickSet(bs, dims, _bitmap=(bitmap, tiles, P, nb))
    out._grid = grid  # C-order brick bits, when the vote produced them
    return out


class Lbvh:
    """Node-array BVH (lbvh.py:105-144): internal rows 0..n-2 then the n leaves in Morton
    order; ``left``/``right`` -1 on leaves; ``leaf_brick`` maps a leaf to its
    ``brick_coords`` row.  Device arrays in ``dev``; host arrays on first access."""

    _FIELDS = ("lo", "hi", "left", "right", "leaf_brick", "brick_coords")

    def __init__(self, dev: dict, info: torch.Tensor, brick_size: int, dims):
        self.dev = dev              # device tensors with capacity rows
        self.info = info            # device int32 {n_bricks, height}
        self.brick_size = int(brick_size)
        self.dims = tuple(int(d) for d in dims)
        self._host = {}
        self._info_host = None

    def _ih(self):
        if self._info_host is None:
            self._info_host = [int(v) for v in self.info.cpu().tolist()]
        return self._info_host

    @property
    def n_bricks(self) -> int:
        return self._ih()[0]

    @property
    def node_count(self) -> int:
        n = self.n_bricks
        return 2 * n - 1 if n else 0

    @property
    def root(self) -> int:
        return 0 if self.n_bricks else -1

    def height(self) -> int:
        """Nodes on the longest root-to-leaf path (lbvh.py:128-144).  The bitmap builder does
        not climb the tree, so, like the reference's DFS, the height is computed on the first
        call (vs_lbvh_height) and kept in ``info``."""
        h = self._ih()[1]
        if h < 0:
            cap = self.dev["brick_coords"].shape[0]
            wsb = query("vs_lbvh_height_workspace", cap)
            ws = _lib.workspace(wsb)
            call("vs_lbvh_height", ptr(self.dev["left"]), ptr(self.dev["right"]), ptr(self.info),
                 cap, ptr(ws), wsb, stream())
            self._info_host = None
            h = self._ih()[1]
        return h

    def __getattr__(self, name):
        if name in Lbvh._FIELDS:
            h = self.__dict__["_host"]
            if name not in h:
                m = self.node_count
                rows = self.n_bricks if name == "brick_coords" else m
                t = self.dev[name][:rows]
                h[name] = t.cpu().numpy().astype(np.int32, copy=False)
            return h[name]
        raise AttributeError(name)

    def is_leaf(self, i: int) -> bool:
        return self.left[i] < 0

    def brick_grid_dims(self):
        return tuple(-(-d // self.brick_size) for d in self.dims)

    def brick_grid(self) -> torch.Tensor:
        """C-order bit grid of the leaf bricks (renderer's brick DDA), built on first use."""
        g = self.__dict__.get("_brick_grid")
        if g is None:
            nb = self.brick_grid_dims()
            words = (nb[0] * nb[1] * nb[2] + 31) // 32
            g = torch.empty(max(words, 1), dtype=torch.int32, device=self.info.device)
            cap = self.dev["brick_coords"].shape[0]
            call("vs_lbvh_brick_grid", ptr(self.dev["brick_coords"]), ptr(self.info), cap, *nb,
                 ptr(g), stream())
            self.__dict__["_brick_grid"] = g
        return g


def empty_lbvh(brick_size: int, dims) -> Lbvh:
    dev = _lib.device()
    z3 = torch.zeros((1, 3), dtype=torch.int32, device=dev)
    z1 = torch.zeros(1, dtype=torch.int32, device=dev)
    d = {"lo": z3, "hi": z3.clone(), "left": z1, "right": z1.clone(), "leaf_brick": z1.clone(),
         "brick_coords": z3.clone()}
    return Lbvh(d, torch.zeros(2, dtype=torch.int32, device=dev), brick_size, dims)


def _alloc_tree(cap: int, dev) -> dict:
    m = max(2 * cap - 1, 1)
    return {
        "lo": torch.empty((m, 3), dtype=torch.int32, device=dev),
        "hi": torch.empty((m, 3), dtype=torch.int32, device=dev),
        "left": torch.empty(m, dtype=torch.int32, device=dev),
        "right": torch.empty(m, dtype=torch.int32, device=dev),
        "leaf_brick": torch.empty(m, dtype=torch.int32, device=dev),
        "brick_coords": torch.empty((max(cap, 1), 3), dtype=torch.int32, device=dev),
    }


def build_lbvh(bricks: BrickSet) -> Lbvh:
    """Sort bricks by Morton code (ties by scan index), Karras radix tree, refit; leaf boxes
    are brick boxes clipped to dims (lbvh.py:216-264)."""
    bs, dims = bricks.brick_size, bricks.dims
    nx, ny, nz = dims
    dev = _lib.device()
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    if bricks._bitmap is not None:
        bitmap, tiles, P, nb = bricks._bitmap
        cap = nb[0] * nb[1] * nb[2]
        d = _alloc_tree(cap, dev)
        wsb = query("vs_lbvh_workspace", P, cap)
        ws = _lib.workspace(wsb)
        grid = getattr(bricks, "_grid", None)
        fill = grid is None  # the vote did not write the renderer's brick grid: leaves do
        if fill:
            grid = torch.empty(max((cap + 31) // 32, 1), dtype=torch.int32, device=dev)
        call("vs_lbvh_from_bitmap", ptr(bitmap), ptr(tiles), P, bs, nx, ny, nz, cap,
             ptr(d["lo"]), ptr(d["hi"]), ptr(d["left"]), ptr(d["right"]), ptr(d["leaf_brick"]),
             ptr(d["brick_coords"]), ptr(grid) if fill else None, ptr(info), ptr(ws), wsb,
             stream())
        out = Lbvh(d, info, bs, dims)
        out.__dict__["_brick_grid"] = grid
        return out
    n = bricks.count
    if n == 0:
        return empty_lbvh(bs, dims)
    coords = torch.from_numpy(np.ascontiguousarray(bricks.coords, dtype=np.int32)).to(dev)
    codes = torch.from_numpy(np.ascontiguousarray(bricks.codes, dtype=np.uint32).view(np.int32)).to(dev)
    d = _alloc_tree(n, dev)
    wsb = query("vs_lbvh_bricks_workspace", n)
    ws = _lib.workspace(wsb)
    call("vs_lbvh_from_bricks", ptr(coords), ptr(codes), n, bs, nx, ny, nz, ptr(d["lo"]),
         ptr(d["hi"]), ptr(d["left"]), ptr(d["right"]), ptr(d["leaf_brick"]),
         ptr(d["brick_coords"]), ptr(info), ptr(ws), wsb, stream())
    return Lbvh(d, info, bs, dims)


def leaf_boxes(idx: Lbvh) -> list[Aabb]:
    out = []
    left, lo, hi = idx.left, idx.lo, idx.hi
    for i in range(idx.node_count):
        if left[i] < 0:
            out.append(Aabb(tuple(int(c) for c in lo[i]), tuple(int(c) for c in hi[i])))
    return out
