"""Macro-cell grid (and, later in this module, summed-volume tables) on the B200.

Drop-in for voxelskip.svt (/root/reference/pkg/src/voxelskip/svt.py).  derive_macro_grid on a
lazy classification with 16^3 cells reuses the fused brick summary (a 16-cell is the OR of its
2x2x2 aligned 8-bricks), otherwise it votes over the packed bits (vs_vote_cells).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, stream
from .volume import BinaryVolume

DEFAULT_BRICK_SIZE = 32


class MacroGrid:
    """Coarse occupancy grid (svt.py:29-37): ``occupied`` is (ncx, ncy, ncz) bool.

    Same constructor as the reference dataclass -- ``MacroGrid(cell_size, cells_dims, dims,
    occupied)`` -- where ``occupied`` may be a host bool array (uploaded on first render) or
    the device uint8 tensor the builders produce (read back on first host access)."""

    def __init__(self, cell_size: int, cells_dims, dims, occupied):
        self.cell_size = int(cell_size)
        self.cells_dims = tuple(int(c) for c in cells_dims)
        self.dims = tuple(int(d) for d in dims)
        if isinstance(occupied, torch.Tensor):
            self._dev, self._host = occupied, None
        else:
            host = np.ascontiguousarray(occupied, dtype=bool)
            if host.shape != self.cells_dims:
                raise ValueError(f"occupied has shape {host.shape}, cells_dims {self.cells_dims}")
            self._dev, self._host = None, host

    @property
    def occupied(self) -> np.ndarray:
        if self._host is None:
            self._host = self._dev.cpu().numpy().view(bool)
        return self._host

    @property
    def occupied_dev(self) -> torch.Tensor:
        """uint8 (ncx, ncy, ncz) on the device."""
        if self._dev is None:
            self._dev = torch.from_numpy(self._host.view(np.uint8).copy()).to(_lib.device())
        return self._dev

    def storage_bytes(self) -> int:
        return (int(np.prod(self.cells_dims)) + 7) // 8  # packbits size, as svt.py:36-37


def derive_macro_grid(source, cell_size: int) -> MacroGrid:
    """A cell is occupied iff it holds >= 1 set flag; border cells clipped (svt.py:134-167)."""
    if cell_size < 2:
        raise ValueError("cell_size must be >= 2")
    cs = int(cell_size)
    b = source if isinstance(source, BinaryVolume) else getattr(source, "binary", None)
    if b is None:
        raise TypeError("derive_macro_grid needs a BinaryVolume or an SvtGrid")
    dims = b.dims
    nx, ny, nz = dims
    nc = tuple(-(-d // cs) for d in dims)
    dev = _lib.device()
    occ = torch.empty(nc, dtype=torch.uint8, device=dev)
    if cs == 16 and b.lazy and b.summary_ok():
        nb = tuple(-(-d // 8) for d in dims)
        P = query("vs_morton_side", *nb)
        bitmap = torch.empty(P * P * P // 32, dtype=torch.int32, device=dev)
        tiles = torch.empty(P * P * P // 512, dtype=torch.int32, device=dev)
        b.vote_bitmap(P, bitmap, tiles, cell16=occ)
    else:
        call("vs_vote_cells", ptr(b.packed()), nx, ny, nz, cs, ptr(occ), stream())
    return MacroGrid(cs, nc, dims, occ)


class SvtGrid:
    """Per-brick summed-volume tables (svt.py:20-26) over a classification.

    ``tables`` (nbx, nby, nbz, bs+1, bs+1, bs+1) uint32 is built on the device on first use
    (vs_svt_build); the k-d builders read the packed bits directly, so a TF-change k-d
    rebuild never pays for the tables unless they are asked for."""

    def __init__(self, b: BinaryVolume, brick_size: int):
        self.binary = b
        self.brick_size = int(brick_size)
        self.dims = b.dims
        self.bricks_dims = tuple(-(-d // self.brick_size) for d in self.dims)
        self._tables_dev = None
        self._tables = None

    @property
    def bits(self) -> np.ndarray:
        return self.binary.bits

    def tables_dev(self) -> torch.Tensor:
        if self._tables_dev is None:
            nb, e = self.bricks_dims, self.brick_size + 1
            t = torch.empty((*nb, e, e, e), dtype=torch.int32, device=_lib.device())
            nx, ny, nz = self.dims
            call("vs_svt_build", ptr(self.binary.packed()), nx, ny, nz, self.brick_size, ptr(t),
                 stream())
            self._tables_dev = t
        return self._tables_dev

    @property
    def tables(self) -> np.ndarray:
        if self._tables is None:
            self._tables = self.tables_dev().cpu().numpy().view(np.uint32)
        return self._tables


def build_svt_grid(b: BinaryVolume, brick_size: int = DEFAULT_BRICK_SIZE) -> SvtGrid:
    """Cumulative-count tables for every brick (svt.py:40-57); built lazily on the device."""
    if brick_size < 2:
        raise ValueError("brick_size must be >= 2")
    if brick_size > 32:
        raise ValueError("brick_size > 32 is not supported by the device table builder")
    return SvtGrid(b, brick_size)


def box_count(g: SvtGrid, box) -> int:
    """Exact number of set flags inside ``box`` (svt.py:65-90), from the tables."""
    t = g.tables_dev()
    dev = t.device
    b = torch.tensor([list(box.lo) + list(box.hi)], dtype=torch.int32, device=dev)
    out = torch.zeros(1, dtype=torch.int64, device=dev)
    nx, ny, nz = g.dims
    call("vs_box_count", ptr(t), nx, ny, nz, g.brick_size, ptr(b), 1, ptr(out), stream())
    return int(out.item())


def tight_box(b: BinaryVolume, box):
    """Minimal box holding every flag of ``box`` (None when empty), from the packed bits."""
    from .volume import Aabb

    dev = _lib.device()
    bx = torch.tensor(list(box.lo) + list(box.hi), dtype=torch.int32, device=dev)
    out = torch.empty(6, dtype=torch.int32, device=dev)
    nx, ny, nz = b.dims
    call("vs_tight_box", ptr(b.packed()), nx, ny, nz, ptr(bx), ptr(out), stream())
    r = out.cpu().tolist()
    if r[3] < 0:
        return None
    return Aabb(tuple(r[:3]), tuple(r[3:]))


def shrink_to_occupied(g: SvtGrid, box):
    """Minimal box containing every set flag inside ``box``, or None (svt.py:100-131)."""
    return tight_box(g.binary, box)
