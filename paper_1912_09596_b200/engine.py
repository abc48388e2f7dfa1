"""Resident TF-change rebuild engines (the interactive "per-frame rebuild on a TF sweep" path).

``LbvhRebuilder`` owns every device buffer of one volume's LBVH rebuild (summary, Morton
bitmap, tile counts, tree arrays, workspace) so a rebuild is a fixed launch sequence:

    cold: vs_classify_summary -> vs_summary_to_bitmap -> vs_lbvh_from_bitmap
    warm: vs_presence_to_bitmap -> vs_lbvh_from_bitmap   (per-volume presence masks, built
          once: a TF change reads 32 B per brick instead of the volume)

reading the TF only through a 64-byte device parameter block.  The sequence is captured once
into a CUDA graph; a TF change is then one 64-byte copy + one graph launch, with the index
(and its brick count / height) ready on the device and no host synchronisation.
The results are the same arrays build_lbvh(flag_bricks(classify(v, tf, dilate=True))) returns.
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import call, ptr, query
from .lbvh import Lbvh, _alloc_tree
from .svt import MacroGrid
from .volume import TransferFunction, Volume, presence_table


class LbvhRebuilder:
    """``v`` is one Volume or a list of up to 4 channels (multichannel.py semantics: the
    hierarchy covers the union of the channels' visible voxels; one 64-byte TF block per
    channel, stacked)."""

    def __init__(self, v, brick_size: int = 8, with_grid: bool = False, count: bool = False,
                 warm: bool = False):
        self.channels = list(v) if isinstance(v, (list, tuple)) else [v]
        v = self.channels[0]
        if brick_size != 8 or v.dims[2] % 16 != 0:
            raise ValueError("LbvhRebuilder needs 8^3 bricks and nz % 16 == 0")
        if len(self.channels) > 1 and count:
            raise ValueError("count is single-channel only")
        if warm and count:
            raise ValueError("the warm rebuild does not read the volume: no voxel count")
        self.warm = bool(warm)
        self.v = v
        self.dims = v.dims
        nx, ny, nz = v.dims
        dev = _lib.device()
        self.nb = tuple(-(-d // 8) for d in v.dims)
        self.P = query("vs_morton_side", *self.nb)
        self.cap = self.nb[0] * self.nb[1] * self.nb[2]
        self.params = torch.zeros(16 * len(self.channels), dtype=torch.int32, device=dev)
        self.summary_tmp = torch.empty(self.cap, dtype=torch.int32, device=dev) \
            if len(self.channels) > 1 else None
        self.summary = torch.empty(self.cap, dtype=torch.int32, device=dev)
        self.bitmap = torch.empty(self.P ** 3 // 32, dtype=torch.int32, device=dev)
        self.tiles = torch.empty(self.P ** 3 // 512, dtype=torch.int32, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev) if count else None
        self.grid = None
        if with_grid:
            nc = tuple(-(-d // 16) for d in v.dims)
            self.grid = torch.empty(nc, dtype=torch.uint8, device=dev)
        self.tree = _alloc_tree(self.cap, dev)
        self.info = torch.zeros(2, dtype=torch.int32, device=dev)
        self.wsb = query("vs_lbvh_workspace", self.P, self.cap)
        self.ws = torch.empty(self.wsb, dtype=torch.uint8, device=dev)
        words = (self.cap + 31) // 32
        self.brick_bits = torch.empty(max(words, 1), dtype=torch.int32, device=dev)
        self.presence = None
        if self.warm:  # the channels' per-volume halo presence masks (built once per volume)
            self.presence = presence_table(self.channels)
        self.graph = None
        self._view = None

    # -- the launch sequence ------------------------------------------------------------
    def launch_summary(self, st: int):
        nx, ny, nz = self.dims
        if self.warm:
            return  # the presence masks replace the per-TF volume pass
        if self.count is not None:
            self.count.zero_()
        if self.summary_tmp is None:
            call("vs_classify_summary", ptr(self.v.bins), nx, ny, nz, ptr(self.params),
                 ptr(self.summary), None, ptr(self.count), st)
            return
        for c, ch in enumerate(self.channels):  # union of the channels' classifications
            out = self.summary if c == 0 else self.summary_tmp
            call("vs_classify_summary", ptr(ch.bins), nx, ny, nz, ptr(self.params[16 * c:]),
                 ptr(out), None, None, st)
            if c:
                call("vs_or_words", ptr(self.summary), ptr(out), self.cap, st)

    def launch_tree(self, st: int):
        self.launch_vote(st)
        self.launch_build(st)

    def launch_vote(self, st: int):
        """The dilated brick vote into the Morton bitmap (warm: presence masks; cold: summary);
        it also writes the leaf-brick grid for the renderer's brick DDA ("index ready")."""
        nx, ny, nz = self.dims
        if self.warm:
            call("vs_presence_to_bitmap", ptr(self.presence), ptr(self.params),
                 len(self.channels), nx, ny, nz, self.P, ptr(self.bitmap), ptr(self.tiles),
                 ptr(self.grid), ptr(self.brick_bits), st)
        else:
            call("vs_summary_to_bitmap", ptr(self.summary), nx, ny, nz, 1, self.P,
                 ptr(self.bitmap), ptr(self.tiles), ptr(self.grid), ptr(self.brick_bits), st)

    def launch_build(self, st: int):
        nx, ny, nz = self.dims
        t = self.tree
        call("vs_lbvh_from_bitmap", ptr(self.bitmap), ptr(self.tiles), self.P, 8, nx, ny, nz,
             self.cap, ptr(t["lo"]), ptr(t["hi"]), ptr(t["left"]), ptr(t["right"]),
             ptr(t["leaf_brick"]), ptr(t["brick_coords"]), None, ptr(self.info), ptr(self.ws),
             self.wsb, st)

    def launch(self):
        st = torch.cuda.current_stream().cuda_stream
        self.launch_summary(st)
        self.launch_tree(st)

    def capture(self):
        """Capture the rebuild into a CUDA graph (replayed by rebuild())."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.launch()  # warm-up outside capture (CUB / module loading)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch()
        self.graph = g
        return self

    def set_tf(self, tf_params: torch.Tensor):
        """tf_params: device int32[16 * channels] vs_tf_params block(s)."""
        self.params.copy_(tf_params.reshape(-1), non_blocking=True)

    def rebuild(self, tf_params: torch.Tensor | None = None):
        if tf_params is not None:
            self.set_tf(tf_params)
        if self.graph is not None:
            self.graph.replay()
        else:
            self.launch()

    # -- results --------------------------------------------------------------------------
    def index(self) -> Lbvh:
        """A live Lbvh over the rebuilder's buffers (valid until the next rebuild)."""
        if self._view is None:
            v = Lbvh(self.tree, self.info, 8, self.dims)
            v.__dict__["_brick_grid"] = self.brick_bits
            self._view = v
        return self._view

    def lbvh(self) -> Lbvh:
        """A snapshot Lbvh (device arrays cloned) of the last rebuild."""
        d = {k: t.clone() for k, t in self.tree.items()}
        return Lbvh(d, self.info.clone(), 8, self.dims)

    def macro_grid(self) -> MacroGrid:
        nc = tuple(-(-d // 16) for d in self.dims)
        return MacroGrid(16, nc, self.dims, self.grid.clone())

    def algorithmic_bytes(self, n_bricks: int) -> dict:
        """SURVEY.md §8(d) B_lbvh terms for one rebuild (compulsory traffic only).  The warm
        rebuild replaces the volume read by the presence masks (32 B per brick per channel)."""
        nx, ny, nz = self.dims
        vol = nx * ny * nz
        tree = 16 * n_bricks + 36 * (2 * n_bricks - 1) + 12 * n_bricks
        return {
            "summary_kernel": vol + 4 * self.cap,           # u8 read + 27-bit summary write
            "rebuild": vol + tree,                          # B_lbvh (cold)
            "rebuild_warm": 32 * self.cap * len(self.channels) + tree,
        }


def tf_params_device(tfs: list[TransferFunction]) -> torch.Tensor:
    """Stack of vs_tf_params blocks for a TF sweep, resident on the device."""
    import numpy as np

    host = np.stack([tf.params_host() for tf in tfs])
    return _lib.upload(host)
