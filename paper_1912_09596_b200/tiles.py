"""Image-tile parallel rendering across GPUs: one process per GPU, the volume
and the index replicated on every rank, the frame split into interleaved row stripes
(stripe rows dealt round-robin over the ranks, which balances the volume's central
footprint), each rank renders its stripes with k_render, and the RGBA8 stripes are gathered
over NVLink with one NCCL all-gather, then put back in image order.

World size 1 renders the whole frame with no collective.  The same code path runs on CPU
process groups (gloo) for the host-side tests of the stripe bookkeeping.
"""

from __future__ import annotations

import sys

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .render import (Camera, Frame, RenderTarget, RowsDesc, _check_flag_bits, _check_flags,
                     camera_desc,
                     index_desc, render_rows, volume_desc)

DEFAULT_STRIPE = 8


def stripe_rows(height: int, nparts: int, part: int, stripe: int = DEFAULT_STRIPE) -> np.ndarray:
    """Image rows rendered by ``part``: stripes of ``stripe`` rows dealt round-robin."""
    rows = np.arange(height)
    return rows[(rows // stripe) % nparts == part]


def gather_permutation(height: int, nparts: int, stripe: int = DEFAULT_STRIPE):
    """(max local rows, index array mapping gathered (part, local row) slots -> image rows)."""
    per = [stripe_rows(height, nparts, p, stripe) for p in range(nparts)]
    mx = max(len(r) for r in per)
    src = np.empty(height, dtype=np.int64)
    for p, r in enumerate(per):
        src[r] = p * mx + np.arange(len(r))
    return mx, src


def assemble(gathered: torch.Tensor, perm: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """Gathered (world*maxrows, w, 4) stripe slots -> image rows (out[j] = gathered[perm[j]])."""
    return torch.index_select(gathered, 0, perm, out=out)


def presence_slabs(nbx: int, nparts: int) -> list[tuple[int, int]]:
    """Brick x-slab range [bx0, bx1) of each part for the sharded presence build: equal
    ceil(nbx / nparts) slabs per part (the last ones short or empty), so every rank's slice
    of the all-gather has the same size."""
    per = -(-nbx // nparts)
    return [(min(nbx, p * per), min(nbx, (p + 1) * per)) for p in range(nparts)]


def shard_presence(v, group=None, builder=None) -> torch.Tensor:
    """The volume's per-brick halo presence masks (Volume.presence, vs_presence_build) built
    sharded over a process group: rank r builds its brick x-slabs of the replicated volume
    (vs_presence_build_slab) and one all-gather (NCCL over NVLink on device buffers; host
    copies for a gloo group) assembles the array on every rank.  Bit-identical to the
    single-GPU build (the slabs are independent: each brick reads only its own halo).
    World size 1 is the plain build.  ``builder(bx0, bx1, out)`` overrides the slab build
    (CPU-side tests of the split)."""
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    nx, ny, nz = v.dims if hasattr(v, "dims") else v._dims
    nbx, nby, nbz = -(-nx // 8), -(-ny // 8), -(-nz // 8)
    slab_words = nby * nbz * 8
    if world == 1 and builder is None:
        return v.presence()
    rank = dist.get_rank(group) if world > 1 else 0
    per = -(-nbx // world)
    dev = v.bins.device if builder is None else torch.device("cpu")
    full = torch.zeros(world * per * slab_words, dtype=torch.int32, device=dev)
    bx0, bx1 = presence_slabs(nbx, world)[rank]
    mine = full[rank * per * slab_words: (rank + 1) * per * slab_words]
    if builder is not None:
        builder(bx0, bx1, mine)
    elif bx1 > bx0:
        # the slab kernel writes at the slab's offset of a full-size array: point it at
        # ``mine`` shifted back by bx0 slabs (only words of [bx0, bx1) are written)
        base = mine.data_ptr() - bx0 * slab_words * 4
        _lib.call("vs_presence_build_slab", _lib.ptr(v.bins), nx, ny, nz, bx0, bx1, base,
                  _lib.stream())
    if world > 1:
        local = mine.clone()
        if dev.type == "cuda" and dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(full, local, group=group)
        else:
            host = torch.empty(full.shape, dtype=full.dtype)
            dist.all_gather_into_tensor(host, local.cpu(), group=group)
            full.copy_(host)
    p = full[: nbx * slab_words]
    if builder is None:
        v.__dict__["_presence"] = p  # Volume.presence() returns the assembled array
        v.__dict__.pop("_presence_tab", None)
    return p


class TileRenderer:
    """Renders frames of one (volume, index) with the rows split over a process group."""

    def __init__(self, width: int, height: int, group=None, stripe: int = DEFAULT_STRIPE,
                 want_samples: bool = False):
        self.width, self.height = int(width), int(height)
        self.group = group
        self.world = dist.get_world_size(group) if (dist.is_available() and
                                                    dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.stripe = int(stripe)
        self.rows = stripe_rows(self.height, self.world, self.rank, self.stripe)
        self.maxrows, perm = gather_permutation(self.height, self.world, self.stripe)
        dev = _lib.device()
        self.target = RenderTarget(self.width, self.maxrows, want_samples=want_samples)
        self.rows_desc = RowsDesc(len(self.rows), self.stripe, self.world, self.rank)
        if self.world > 1:
            self.gathered = torch.empty((self.world * self.maxrows, self.width, 4),
                                        dtype=torch.uint8, device=dev)
            self.totals = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.perm = torch.from_numpy(perm).to(dev)
        self.frame_dev = torch.empty((self.height, self.width, 4), dtype=torch.uint8, device=dev)

    def render(self, v, tf, index, cam: Camera, dt: float = 0.5, idx_desc=None, vol_desc=None,
               cam_desc=None, ert_eps: float = 0.0) -> torch.Tensor:
        """Render this rank's stripes and assemble the full frame on every rank (device).
        ``ert_eps`` > 0: opt-in early ray termination (RGBA within ert_eps of the reference
        integral, fewer samples); 0 is the reference's integrator."""
        self._last_total = self.target.total
        render_rows(v, tf, index, cam, self.target, dt=dt, rows=self.rows_desc,
                    idx_desc=idx_desc or index_desc(index), vol_desc=vol_desc or volume_desc(v),
                    cam_desc=cam_desc or camera_desc(cam), ert_eps=ert_eps)
        if self.world == 1:
            self.frame_dev.copy_(self.target.rgba8[: self.height])
            return self.frame_dev
        self._gather(self.target.rgba8)
        return assemble(self.gathered, self.perm, self.frame_dev)

    def _gather(self, local: torch.Tensor):
        """All-gather of the equal-size stripe sets: NCCL over NVLink on device buffers; a gloo
        group (CPU-side tests of the split) goes through host copies."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self.gathered, local, group=self.group)
        else:
            host = torch.empty(self.gathered.shape, dtype=self.gathered.dtype)
            dist.all_gather_into_tensor(host, local.cpu(), group=self.group)
            self.gathered.copy_(host)

    def render_multi(self, volumes, tfs, index, cam: Camera, dt: float = 0.5,
                     checked: bool = True) -> torch.Tensor:
        """Multi-channel frame (multichannel.py), same stripe split and gather.  ``checked``
        verifies the segment capacity (one synchronisation, re-render on overflow); unchecked
        frames queue without a host sync and accumulate RF_SEGCAP in ``multi_flags()``."""
        from .multichannel import MultiTarget, render_multi_checked, render_multi_rows

        mt = self.__dict__.get("_multi_target")
        if mt is None:
            mt = MultiTarget(self.width, self.maxrows)
            self._multi_target = mt
        if checked:
            render_multi_checked(volumes, tfs, index, cam, mt, dt, rows=self.rows_desc)
        else:
            mt.total.zero_()
            render_multi_rows(volumes, tfs, index, cam, mt, dt, rows=self.rows_desc, zero=False)
        self._last_total = mt.total
        if self.world == 1:
            self.frame_dev.copy_(mt.rgba8[: self.height])
            return self.frame_dev
        self._gather(mt.rgba8)
        return assemble(self.gathered, self.perm, self.frame_dev)

    def multi_flags(self) -> int:
        """Renderer flags accumulated by unchecked multi-channel frames since the last read."""
        mt = self.__dict__.get("_multi_target")
        if mt is None:
            return 0
        f = int(mt.flags.item())
        mt.flags.zero_()
        return f

    def sample_total(self) -> int:
        t = self.__dict__.get("_last_total", self.target.total)
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(self.totals, t, group=self.group)
                return int(self.totals.sum().item())
            host = torch.empty(self.world, dtype=torch.int64)
            dist.all_gather_into_tensor(host, t.cpu(), group=self.group)
            return int(host.sum())
        return int(t.item())

    def frame(self, v, tf, index, cam: Camera, dt: float = 0.5) -> Frame:
        """Public API: a full Frame (host pixels) rendered by the whole group.

        Pixels, the renderer's flags and the sample total come back in one asynchronous copy
        into pinned host memory.  The Frame's pixel array IS the pinned buffer; it is recycled
        for a later frame only once the caller has dropped every reference to it (otherwise a
        fresh pinned buffer is allocated)."""
        return self.frame_async(v, tf, index, cam, dt).result()

    def frame_async(self, v, tf, index, cam: Camera, dt: float = 0.5) -> "PendingFrame":
        """Render now; the readback runs on a copy stream so the next frame's work can be
        queued while this one travels to the host.  ``.result()`` waits and returns the Frame."""
        img = self.render(v, tf, index, cam, dt)
        return self._readback(img, self.target.flags)

    def frame_multi_async(self, volumes, tfs, index, cam: Camera,
                          dt: float = 0.5) -> "PendingFrame":
        """frame_async for a multi-channel volume (capacity-checked render_multi)."""
        img = self.render_multi(volumes, tfs, index, cam, dt)
        return self._readback(img, self._multi_target.flags)

    def _readback(self, img: torch.Tensor, flags: torch.Tensor) -> "PendingFrame":
        total = self._last_total
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(self.totals, total, group=self.group)
                total = self.totals.sum().reshape(1)
            else:
                total = torch.tensor([self.sample_total()], dtype=torch.int64, device=img.device)
        slot = self._free_slot(img)
        cur = torch.cuda.current_stream()
        # device-side snapshot (the next render reuses frame_dev), then the D2H on the copy stream
        slot["dev"].copy_(img)
        slot["meta_dev"][0].copy_(flags.to(torch.int64).reshape(()))
        slot["meta_dev"][1].copy_(total.reshape(()))
        cs = self.__dict__.setdefault("_copy_stream", torch.cuda.Stream())
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            slot["t"].copy_(slot["dev"], non_blocking=True)
            slot["meta"].copy_(slot["meta_dev"], non_blocking=True)
            slot["done"].record(cs)
        slot["busy"] = True
        return PendingFrame(self, slot)

    def _free_slot(self, img: torch.Tensor) -> dict:
        ring = self.__dict__.setdefault("_pinned_ring", [])
        for s in ring:
            # free when not pending and only the ring entry (and getrefcount's argument)
            # refers to its pixel array
            if not s["busy"] and sys.getrefcount(s["pixels"]) <= 2:
                return s
        pix = torch.empty(img.shape, dtype=img.dtype).pin_memory()
        slot = {"t": pix, "pixels": pix.numpy(), "dev": torch.empty_like(img),
                "meta": torch.empty(2, dtype=torch.int64).pin_memory(),
                "meta_dev": torch.empty(2, dtype=torch.int64, device=img.device),
                "done": torch.cuda.Event(), "busy": False}
        ring.append(slot)
        return slot


class PendingFrame:
    """A frame whose pixels are on their way to pinned host memory (TileRenderer.frame_async)."""

    def __init__(self, tr: TileRenderer, slot: dict):
        self._tr, self._slot, self._frame = tr, slot, None

    def result(self) -> Frame:
        if self._frame is None:
            s = self._slot
            s["done"].synchronize()
            flags, samples = (int(x) for x in s["meta"].tolist())
            s["busy"] = False
            _check_flag_bits(flags)
            self._frame = Frame(width=self._tr.width, height=self._tr.height,
                                pixels=s["pixels"], sample_count=samples)
        return self._frame
