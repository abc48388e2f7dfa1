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
    """Coarse occupancy grid (svt.py:29-37): ``occupied`` is (ncx, ncy, ncz) bool."""

    def __init__(self, cell_size: int, cells_dims, dims, occupied_dev: torch.Tensor):
        self.cell_size = int(cell_size)
        self.cells_dims = tuple(int(c) for c in cells_dims)
        self.dims = tuple(int(d) for d in dims)
        self.occupied_dev = occupied_dev  # uint8 (ncx, ncy, ncz) on the device
        self._host = None

    @property
    def occupied(self) -> np.ndarray:
        if self._host is None:
            self._host = self.occupied_dev.cpu().numpy().view(bool)
        return self._host

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
        call("vs_summary_to_bitmap", ptr(b.summary()), nx, ny, nz, int(b._source[2]), P,
             ptr(bitmap), ptr(tiles), ptr(occ), stream())
    else:
        call("vs_vote_cells", ptr(b.packed()), nx, ny, nz, cs, ptr(occ), stream())
    return MacroGrid(cs, nc, dims, occ)
