"""Multi-channel volumes (BASELINE.json configs[4]): K <= 4 co-registered u8 channels, one TF
per channel, one shared skipping hierarchy.

The reference has no multi-channel path (SPEC.md:125 lists it as a non-goal), so these
semantics are this build's, chosen to reduce exactly to the reference when all channels but
one have zero alpha (the parity anchor, tested against the golden single-channel frames):

* classification: a voxel is visible iff any channel's TF gives it alpha > 0; dilation and
  brick votes follow on the union (the brick summary of a union is the OR of summaries);
* compositing: at each lattice sample the channels are composited in channel order with the
  reference's update (w = (1 - A) corr_c; C += w rgb_c; A += w) for every visible channel.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .render import (Camera, Frame, RowsDesc, _check_flags, camera_desc, index_desc, tf_device,
                     volume_desc)
from .volume import BinaryVolume, TransferFunction, Volume, _nzw, presence_table


class MultiBinaryVolume(BinaryVolume):
    """Lazy union classification of several channels."""

    def __init__(self, volumes, tfs, dilate: bool):
        super().__init__(_source=(tuple(volumes), tuple(tfs), bool(dilate)), dims=volumes[0].dims)

    def summary_ok(self) -> bool:
        return self._dims[2] % 16 == 0

    def summary(self, count: bool = False) -> torch.Tensor:
        if self._summary is None:
            vols, tfs, _ = self._source
            nx, ny, nz = self._dims
            nb = [-(-d // 8) for d in self._dims]
            dev = _lib.device()
            acc = torch.zeros(nb[0] * nb[1] * nb[2], dtype=torch.int32, device=dev)
            tmp = torch.empty_like(acc)
            for v, tf in zip(vols, tfs):
                call("vs_classify_summary", ptr(v.bins), nx, ny, nz, ptr(tf.params()), ptr(tmp),
                     None, None, stream())
                call("vs_or_words", ptr(acc), ptr(tmp), acc.numel(), stream())
            self._summary = acc
        return self._summary

    def vote_bitmap(self, P, bitmap, tiles, cell16=None, grid=None):
        """Brick vote of the union: warm (channels seen before with another TF set) from the
        channels' presence masks in one pass, else from the OR of the channels' summaries."""
        vols, tfs, dilate = self._source
        nx, ny, nz = self._dims
        warm = dilate and self._summary is None and len(vols) <= 4 and \
            all([v._warm_vote() for v in vols])
        if warm:
            # the channel pointer table, cached on the first channel per channel tuple (as
            # interleaved_quads caches its volume)
            cache = vols[0].__dict__.setdefault("_presence_tabs", {})
            key = tuple(id(v) for v in vols)
            hit = cache.get(key)
            if hit is None or not all(a is b for a, b in zip(hit[0], vols)):
                hit = (tuple(vols), presence_table(vols))
                cache[key] = hit
            params = torch.cat([tf.params() for tf in tfs])
            call("vs_presence_to_bitmap", ptr(hit[1]), ptr(params), len(vols), nx, ny, nz, P,
                 ptr(bitmap), ptr(tiles), ptr(cell16), ptr(grid), stream())
        else:
            call("vs_summary_to_bitmap", ptr(self.summary()), nx, ny, nz, int(dilate), P,
                 ptr(bitmap), ptr(tiles), ptr(cell16), ptr(grid), stream())

    def packed(self) -> torch.Tensor:
        if self._packed is None:
            vols, tfs, dilate = self._source
            nx, ny, nz = self._dims
            dev = _lib.device()
            base = torch.zeros(nx * ny * _nzw(nz), dtype=torch.int32, device=dev)
            tmp = torch.empty_like(base)
            for v, tf in zip(vols, tfs):
                call("vs_classify_bits", ptr(v.bins), nx, ny, nz, ptr(tf.params()), ptr(tmp), None,
                     stream())
                call("vs_or_words", ptr(base), ptr(tmp), base.numel(), stream())
            if dilate:
                out = torch.empty_like(base)
                call("vs_dilate_bits", ptr(base), nx, ny, nz, ptr(out), stream())
                base = out
            self._packed = base
        return self._packed

    def base_count(self) -> int:
        vols, tfs, _ = self._source
        undilated = MultiBinaryVolume(vols, tfs, False)
        return undilated.count_nonzero()

    def count_nonzero(self) -> int:
        p = self.packed()
        nx, ny, nz = self._dims
        cnt = torch.zeros(1, dtype=torch.int64, device=p.device)
        call("vs_count_bits", ptr(p), nx, ny, nz, ptr(cnt), stream())
        return int(cnt.item())


def classify_multi(volumes, tfs, dilate: bool = False) -> MultiBinaryVolume:
    if len(volumes) != len(tfs) or not 1 <= len(volumes) <= 4:
        raise ValueError("need 1..4 channels with one transfer function each")
    dims = volumes[0].dims
    if any(v.dims != dims for v in volumes):
        raise ValueError("channels must share dims")
    if any(v.field is not None for v in volumes):
        raise ValueError("multi-channel rendering needs 8-bit channels")
    return MultiBinaryVolume(volumes, tfs, dilate)


class MultiDesc(C.Structure):
    _fields_ = [("nch", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("quads", C.c_void_p * 4), ("lut", C.c_void_p * 4), ("corr", C.c_void_p * 4),
                ("mquads", C.c_void_p)]


def interleaved_quads(volumes) -> torch.Tensor:
    """Channel-interleaved trilinear gather volume of the channels (vs_build_mquads), built once
    per channel tuple and cached on the first channel."""
    cache = volumes[0].__dict__.setdefault("_mquads", {})
    key = tuple(id(v) for v in volumes)
    hit = cache.get(key)
    if hit is not None and all(a is b for a, b in zip(hit[0], volumes)):
        return hit[1]
    nx, ny, nz = volumes[0].dims
    size = _lib.query("vs_mquads_size", len(volumes), nx, ny, nz)
    q = torch.empty(size, dtype=torch.int32, device=volumes[0].bins.device)
    bins = (C.c_void_p * 4)(*[ptr(v.bins) for v in volumes])
    call("vs_build_mquads", C.addressof(bins), len(volumes), nx, ny, nz, ptr(q), stream())
    cache[key] = (tuple(volumes), q)
    return q


RF_SEGCAP = 4  # a ray had more lattice ranges than the target's segment capacity


class MultiTarget:
    def __init__(self, width: int, nrows: int, cap: int = 64, want_rgba64=False,
                 want_samples=False):
        dev = _lib.device()
        self.width, self.nrows, self.cap = width, nrows, cap
        self.segs = torch.empty((cap, nrows * width, 2), dtype=torch.int32, device=dev)
        self.counts = torch.empty(nrows * width, dtype=torch.int32, device=dev)
        self.rgba8 = torch.empty((nrows, width, 4), dtype=torch.uint8, device=dev)
        self.rgba64 = torch.empty((nrows, width, 4), dtype=torch.float64, device=dev) \
            if want_rgba64 else None
        self.samples = torch.empty((nrows, width), dtype=torch.int32, device=dev) \
            if want_samples else None
        self.total = torch.zeros(1, dtype=torch.int64, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)


def render_multi_rows(volumes, tfs, index, cam: Camera, target: MultiTarget, dt: float = 0.5,
                      rows: RowsDesc | None = None, zero: bool = True):
    """Launch the multi-channel render into ``target`` (async, no host synchronisation).  A ray
    with more lattice ranges than ``target.cap`` sets RF_SEGCAP in ``target.flags`` and is left
    unintegrated; render_multi_checked re-renders with a larger capacity."""
    if zero:
        target.total.zero_()
        target.flags.zero_()
    md = MultiDesc()
    md.nch = len(volumes)
    md.nx, md.ny, md.nz = volumes[0].dims
    keep = []
    for c, (v, tf) in enumerate(zip(volumes, tfs)):
        lut, corr = tf_device(tf, dt)
        keep += [lut, corr]
        md.lut[c] = ptr(lut)
        md.corr[c] = ptr(corr)
    md.mquads = ptr(interleaved_quads(volumes))
    vd = volume_desc(volumes[0], quads=False)
    idx = index_desc(index)
    cd = camera_desc(cam)
    rp = None if rows is None else C.addressof(rows)
    call("vs_render_segments", C.addressof(vd), C.addressof(idx), C.addressof(cd), float(dt), rp,
         ptr(target.segs), ptr(target.counts), target.cap, ptr(target.flags), None, stream())
    call("vs_render_multi_integrate", C.addressof(md), C.addressof(cd), float(dt), rp,
         ptr(target.segs), ptr(target.counts), target.cap, ptr(target.rgba8), ptr(target.rgba64),
         ptr(target.samples), ptr(target.total), ptr(target.flags), stream())
    del keep


def render_multi_checked(volumes, tfs, index, cam: Camera, target: MultiTarget, dt: float = 0.5,
                         rows: RowsDesc | None = None) -> MultiTarget:
    """render_multi_rows + the capacity check (one synchronisation); on overflow the target
    grows to the frame's largest range count and the frame is rendered again."""
    render_multi_rows(volumes, tfs, index, cam, target, dt, rows)
    if int(target.flags.item()) & RF_SEGCAP:
        need = int(target.counts.max().item())
        fresh = MultiTarget(target.width, target.nrows, cap=need,
                            want_rgba64=target.rgba64 is not None,
                            want_samples=target.samples is not None)
        target.__dict__.update(fresh.__dict__)
        render_multi_rows(volumes, tfs, index, cam, target, dt, rows)
    return target


def render_frame_multi(volumes, tfs, index, cam: Camera, dt: float = 0.5) -> Frame:
    """A frame of a multi-channel volume through a shared index."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    tgt = MultiTarget(cam.width, cam.height)
    render_multi_checked(volumes, tfs, index, cam, tgt, dt)
    _check_flags(tgt.flags)
    return Frame(width=cam.width, height=cam.height, pixels=tgt.rgba8.cpu().numpy(),
                 sample_count=int(tgt.total.item()))


def render_float_multi(volumes, tfs, index, cam: Camera, dt: float = 0.5,
                       rows: RowsDesc | None = None):
    """(float64 RGBA, per-pixel samples) of the frame, or of a row band / stripe set."""
    nrows = cam.height if rows is None else rows.nrows
    tgt = MultiTarget(cam.width, nrows, want_rgba64=True, want_samples=True)
    render_multi_checked(volumes, tfs, index, cam, tgt, dt, rows)
    _check_flags(tgt.flags)
    return tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy().astype(np.int64)
