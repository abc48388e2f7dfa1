"""Scalar volumes, transfer functions and binary classification on the B200.

Drop-in for voxelskip.volume (/root/reference/pkg/src/voxelskip/volume.py): same class and
function names, argument meanings and exceptions.  The data live on the GPU:

* ``Volume`` holds the LUT bins as uint8 (quantize_scalar, volume.py:159-162, is applied once
  at upload; it is the identity on 8-bit data) and, only when the float field is not exactly
  ``f32(bin/255)``, the float32 field the renderer interpolates.  ``.data`` is a lazy host view.
* ``BinaryVolume`` is either materialised (packed bits, 1 bit/voxel, z-packed words) or a lazy
  classification ``(volume, tf, dilate)``.  A lazy one feeds flag_bricks / derive_macro_grid
  through the fused one-pass brick-summary kernel, so a TF-change LBVH rebuild reads the
  volume exactly once and never writes the N^3 bit volume.  ``.bits`` materialises on demand.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, stream

LUT_SIZE = 256


class VolumeFormatError(ValueError):
    """Raw file does not match its metadata (size or layout)."""


class UnsupportedFormatError(ValueError):
    """Voxel precision outside the supported 8/16-bit range."""


@dataclass(frozen=True)
class Aabb:
    """Half-open integer voxel box [lo, hi) (volume.py:28-61)."""

    lo: tuple[int, int, int]
    hi: tuple[int, int, int]

    def __post_init__(self):
        object.__setattr__(self, "lo", tuple(int(v) for v in self.lo))
        object.__setattr__(self, "hi", tuple(int(v) for v in self.hi))
        if any(l > h for l, h in zip(self.lo, self.hi)):
            raise ValueError(f"inverted bounds {self.lo}..{self.hi}")

    def volume(self) -> int:
        e = self.extent()
        return e[0] * e[1] * e[2]

    def extent(self) -> tuple[int, int, int]:
        return tuple(h - l for l, h in zip(self.lo, self.hi))

    def contains(self, p) -> bool:
        return all(l <= c < h for l, c, h in zip(self.lo, p, self.hi))

    def union(self, other: "Aabb") -> "Aabb":
        return Aabb(tuple(map(min, self.lo, other.lo)), tuple(map(max, self.hi, other.hi)))

    def intersect(self, other: "Aabb") -> "Aabb | None":
        lo = tuple(map(max, self.lo, other.lo))
        hi = tuple(map(min, self.hi, other.hi))
        if any(l >= h for l, h in zip(lo, hi)):
            return None
        return Aabb(lo, hi)


# f32(u/255) for every u8 (load_raw normalises in float64 then narrows, volume.py:193-194)
U8_FIELD = (np.arange(256, dtype=np.float64) / 255.0).astype(np.float32)


class Volume:
    """Dense scalar field normalised to [0, 1], shape (nx, ny, nz), C-order (volume.py:64-81).

    ``Volume(data)`` follows the reference exactly: ``data`` (numpy or torch, any dtype) is
    cast to float32 (volume.py:70-73) -- a uint8 array therefore holds raw values 0..255, which
    quantise to bin 255 wherever they are nonzero, as in the reference.  8-bit LUT bins (the
    field ``f32(u/255)``, what load_raw returns for 8-bit files) come in through
    ``Volume.from_u8``, which uploads the bytes as they are."""

    def __init__(self, data, name: str = "volume"):
        self._init(data, name, u8_bins=False)

    @classmethod
    def from_u8(cls, bins, name: str = "volume") -> "Volume":
        """8-bit volume whose bytes are the LUT bins (field ``f32(u/255)``, volume.py:193-194).
        ``bins`` must have dtype uint8 (numpy or torch, host or device)."""
        v = cls.__new__(cls)
        v._init(bins, name, u8_bins=True)
        return v

    def _init(self, data, name, u8_bins):
        self.name = name
        dev = _lib.device()
        t = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.asarray(data))
        if t.dim() != 3 or min(t.shape) < 1:
            raise ValueError("volume data must be a non-empty 3-d array")
        self._dims = tuple(int(d) for d in t.shape)
        if u8_bins:
            if t.dtype != torch.uint8:
                raise TypeError(f"Volume.from_u8 needs uint8 bins, got {t.dtype}")
            self.bins = t.to(dev).contiguous()
            self.field = None
        else:
            f = t.to(device=dev, dtype=torch.float32).contiguous()
            bins = torch.empty(self._dims, dtype=torch.uint8, device=dev)
            call("vs_quantize_f32", ptr(f), f.numel(), ptr(bins), stream())
            self.bins = bins
            table = torch.from_numpy(U8_FIELD).to(dev)
            exact = bool(torch.equal(table[bins.long()], f)) if f.numel() <= (1 << 28) else False
            self.field = None if exact else f
        self._host = None

    @property
    def dims(self) -> tuple[int, int, int]:
        return self._dims

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            if self.field is not None:
                self._host = self.field.cpu().numpy()
            else:
                self._host = U8_FIELD[self.bins.cpu().numpy()]
        return self._host

    @property
    def is_u8(self) -> bool:
        return self.field is None

    def quads(self) -> torch.Tensor | None:
        """Trilinear gather volume (4 B/voxel in 4^3 tiles, TF-independent; vs_build_quads),
        built once; None past 2^32 words (the renderer then samples the bins directly)."""
        q = self.__dict__.get("_quads")
        if q is None:
            nx, ny, nz = self._dims
            words = query("vs_quads_words", nx, ny, nz)
            if words >= 1 << 32:
                return None
            q = torch.empty(words, dtype=torch.int32, device=self.bins.device)
            call("vs_build_quads", ptr(self.bins), nx, ny, nz, ptr(q), stream())
            self.__dict__["_quads"] = q
        return q

    def bounds(self) -> Aabb:
        return Aabb((0, 0, 0), self.dims)

    # -- warm path of the brick vote (TF-independent, SURVEY.md §8d cold / warm) -------------
    def presence_ok(self) -> bool:
        return self._dims[2] % 16 == 0 and self.bins.data_ptr() % 16 == 0

    def presence(self) -> torch.Tensor:
        """Per-8^3-brick 256-bit masks of the bins present in the brick's 1-voxel halo
        (vs_presence_build, 32 B per brick), built once per volume.  A dilated brick vote of
        any TF is then (presence & visible bins) != 0 (vs_presence_to_bitmap)."""
        p = self.__dict__.get("_presence")
        if p is None:
            nx, ny, nz = self._dims
            p = torch.empty(query("vs_presence_words", nx, ny, nz), dtype=torch.int32,
                            device=self.bins.device)
            call("vs_presence_build", ptr(self.bins), nx, ny, nz, ptr(p), stream())
            self.__dict__["_presence"] = p
        return p

    def presence_table(self) -> torch.Tensor:
        """Device array holding this volume's presence pointer (vs_presence_to_bitmap's
        channel table for one channel)."""
        t = self.__dict__.get("_presence_tab")
        if t is None:
            t = presence_table([self])
            self.__dict__["_presence_tab"] = t
        return t

    def _warm_vote(self) -> bool:
        """Policy: the first TF on a volume takes the one-pass summary (cold, no extra
        memory); from the second TF on, the presence masks are built once and every later
        dilated vote reads them instead of the volume."""
        if "_presence" in self.__dict__:
            return True
        n = self.__dict__.get("_dilated_votes", 0) + 1
        self.__dict__["_dilated_votes"] = n
        return n >= 2 and self.presence_ok()


class TransferFunction:
    """256-entry RGBA lookup table, all channels in [0, 1] (volume.py:84-140)."""

    def __init__(self, lut):
        self.lut = lut

    @property
    def lut(self) -> np.ndarray:
        return self._lut

    @lut.setter
    def lut(self, lut) -> None:
        """Validated private copy, read-only: the device caches below (params, opacity tables)
        are derived from it, so assigning a new table is the one way to change a TF."""
        lut = np.array(lut, dtype=np.float32, order="C", copy=True)
        if lut.shape != (LUT_SIZE, 4):
            raise ValueError(f"lut must be ({LUT_SIZE}, 4), got {lut.shape}")
        if lut.min() < 0.0 or lut.max() > 1.0:
            raise ValueError("lut channels must lie in [0, 1]")
        lut.setflags(write=False)
        self._lut = lut
        self._dev = {}

    @classmethod
    def constant(cls, r: float, g: float, b: float, a: float) -> "TransferFunction":
        return cls(np.tile(np.array([r, g, b, a], dtype=np.float32), (LUT_SIZE, 1)))

    @classmethod
    def opaque(cls) -> "TransferFunction":
        """Grey, alpha 1 on every bin but 0 (volume.py:102-111)."""
        v = np.linspace(0.0, 1.0, LUT_SIZE, dtype=np.float32)
        a = (np.arange(LUT_SIZE) > 0).astype(np.float32)
        return cls(np.stack([v, v, v, a], axis=1))

    @classmethod
    def ramp(cls, threshold: float = 0.3, max_alpha: float = 0.8,
             color_lo=(0.2, 0.4, 1.0), color_hi=(1.0, 0.6, 0.1)) -> "TransferFunction":
        """Alpha 0 up to ``threshold``, then linear to ``max_alpha`` (volume.py:113-132); the
        colour blends color_lo -> color_hi over the same parameter, computed in float64."""
        v = np.linspace(0.0, 1.0, LUT_SIZE)
        t = np.clip((v - threshold) / max(1e-9, 1.0 - threshold), 0.0, 1.0)
        rgb = (1.0 - t)[:, None] * np.asarray(color_lo)[None, :] + \
            t[:, None] * np.asarray(color_hi)[None, :]
        a = np.where(v > threshold, t * max_alpha, 0.0)
        return cls(np.concatenate([rgb, a[:, None]], axis=1).astype(np.float32))

    @classmethod
    def from_json(cls, path) -> "TransferFunction":
        return cls(np.asarray(json.loads(Path(path).read_text())["rgba"], dtype=np.float32))

    def to_json(self, path) -> None:
        Path(path).write_text(json.dumps({"rgba": self.lut.tolist()}))

    # -- device-side caches -----------------------------------------------------------------
    def params_host(self) -> np.ndarray:
        """vs_tf_params (64 bytes) for this LUT's alpha column."""
        if "params_host" not in self._dev:
            buf = np.zeros(16, dtype=np.int32)
            alpha = np.ascontiguousarray(self.lut[:, 3])
            call("vs_tf_params_from_alpha", alpha.ctypes.data, buf.ctypes.data)
            self._dev["params_host"] = buf
        return self._dev["params_host"]

    def params(self) -> torch.Tensor:
        dev = _lib.device()
        key = ("params", dev.index)
        if key not in self._dev:
            self._dev[key] = _lib.upload(self.params_host())  # 64 bytes, stream-ordered
        return self._dev[key]


def presence_table(volumes) -> torch.Tensor:
    """Device int64 array of the volumes' presence-mask pointers (built on demand)."""
    ptrs = np.array([v.presence().data_ptr() for v in volumes], dtype=np.int64)
    return _lib.upload(ptrs)


def quantize_scalar(values) -> np.ndarray:
    """Host mirror of volume.py:159-162 (floor(v*255 + 0.5) clamped, float64).  The device
    path applies the same rounding in k_quantize."""
    idx = np.floor(np.asarray(values, dtype=np.float64) * 255.0 + 0.5)
    return np.clip(np.nan_to_num(idx, nan=0.0), 0, LUT_SIZE - 1).astype(np.int64)


def _nzw(nz: int) -> int:
    return (nz + 31) // 32


class BinaryVolume:
    """One visibility flag per voxel (volume.py:143-156), held on the GPU.

    ``BinaryVolume(bits)`` packs a host/device bool array.  classify() returns a lazy one
    bound to (volume, tf, dilate)."""

    def __init__(self, bits=None, *, _source=None, dims=None):
        self._packed = None
        self._source = _source
        self._summary = None
        self._count = None
        self._bbox = None  # device int[6] tight box of the flags, when the pack produced it
        self._host = None
        if bits is not None:
            t = bits if isinstance(bits, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(bits), dtype=bool))
            if t.dim() != 3:
                raise ValueError("bits must be 3-d")
            self._dims = tuple(int(d) for d in t.shape)
            dev = _lib.device()
            b8 = t.to(device=dev, dtype=torch.uint8).contiguous()
            nx, ny, nz = self._dims
            self._packed = torch.empty(nx * ny * _nzw(nz), dtype=torch.int32, device=dev)
            if b8.numel():
                call("vs_pack_bits", ptr(b8), nx, ny, nz, ptr(self._packed), stream())
        else:
            self._dims = tuple(int(d) for d in dims)

    @property
    def dims(self) -> tuple[int, int, int]:
        return self._dims

    @property
    def lazy(self) -> bool:
        return self._packed is None

    def summary_ok(self) -> bool:
        """The fused brick-summary kernel applies (8^3 bricks, rows of 16-byte multiples)."""
        return (self._source is not None and self._dims[2] % 16 == 0
                and self._source[0].bins.data_ptr() % 16 == 0)

    def summary(self, count: bool = False) -> torch.Tensor:
        """27-bit halo summaries per 8^3 brick (vs_classify_summary); with ``count`` the
        undilated visible-voxel count is taken in the same pass."""
        if self._summary is None or (count and self._count is None):
            v, tf, _ = self._source
            nx, ny, nz = self._dims
            dev = _lib.device()
            nb = [-(-d // 8) for d in self._dims]
            s = torch.empty(nb[0] * nb[1] * nb[2], dtype=torch.int32, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev) if count else None
            call("vs_classify_summary", ptr(v.bins), nx, ny, nz, ptr(tf.params()), ptr(s), None,
                 ptr(cnt), stream())
            self._summary = s
            if count:
                self._count = cnt
        return self._summary

    def vote_bitmap(self, P: int, bitmap: torch.Tensor, tiles: torch.Tensor,
                    cell16: torch.Tensor | None = None, grid: torch.Tensor | None = None):
        """8^3 brick vote (flag_bricks lbvh.py:83-102; dilated or not) into the Morton bitmap
        + tile counts, optionally the 16^3 macro cells and the C-order leaf-brick bit grid.
        Dilated votes on a volume seen with an earlier TF read its presence masks (warm);
        otherwise the one-pass summary of this classification (cold).  Needs summary_ok()."""
        v, tf, dilate = self._source
        nx, ny, nz = self._dims
        if dilate and self._summary is None and v._warm_vote():
            call("vs_presence_to_bitmap", ptr(v.presence_table()), ptr(tf.params()), 1, nx, ny, nz, P,
                 ptr(bitmap), ptr(tiles), ptr(cell16), ptr(grid), stream())
        else:
            call("vs_summary_to_bitmap", ptr(self.summary()), nx, ny, nz, int(dilate), P,
                 ptr(bitmap), ptr(tiles), ptr(cell16), ptr(grid), stream())

    def packed(self) -> torch.Tensor:
        """Packed bits (int32 words, z-packed rows), materialised on first use."""
        if self._packed is None:
            v, tf, dilate = self._source
            nx, ny, nz = self._dims
            dev = _lib.device()
            base = torch.empty(nx * ny * _nzw(nz), dtype=torch.int32, device=dev)
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            fused = dilate and nz % 32 == 0 and nz <= 1024 and v.bins.data_ptr() % 16 == 0
            if fused:  # the k-d root box comes out of the same pass
                self._bbox = torch.empty(8, dtype=torch.int32, device=dev)
                call("vs_classify_dilate_bits_bbox", ptr(v.bins), nx, ny, nz, ptr(tf.params()),
                     ptr(base), ptr(cnt), ptr(self._bbox), stream())
            else:
                call("vs_classify_bits", ptr(v.bins), nx, ny, nz, ptr(tf.params()), ptr(base),
                     ptr(cnt), stream())
            if self._count is None:
                self._count = cnt
            if dilate and not fused:
                out = torch.empty_like(base)
                call("vs_dilate_bits", ptr(base), nx, ny, nz, ptr(out), stream())
                base = out
            self._packed = base
        return self._packed

    def base_count(self) -> int:
        """Visible voxels of the UNDILATED classification behind a lazy volume."""
        if self._count is None:
            if self.summary_ok():
                self.summary(count=True)
            else:
                self.packed()
        return int(self._count.item())

    def count_nonzero(self) -> int:
        if self._source is not None and not self._source[2]:
            return self.base_count()
        p = self.packed()
        nx, ny, nz = self._dims
        cnt = torch.zeros(1, dtype=torch.int64, device=p.device)
        call("vs_count_bits", ptr(p), nx, ny, nz, ptr(cnt), stream())
        return int(cnt.item())

    @property
    def bits(self) -> np.ndarray:
        if self._host is None:
            p = self.packed()
            nx, ny, nz = self._dims
            out = torch.empty(self._dims, dtype=torch.uint8, device=p.device)
            call("vs_unpack_bits", ptr(p), nx, ny, nz, ptr(out), stream())
            self._host = out.cpu().numpy().view(bool)
        return self._host


def classify(v: Volume, tf: TransferFunction, dilate: bool = False) -> BinaryVolume:
    """Visible iff lut[bin, 3] > 0; with ``dilate`` grown by the clipped 3x3x3 box
    (volume.py:289-319).  Returns a lazy BinaryVolume evaluated by the fused kernels."""
    return BinaryVolume(_source=(v, tf, bool(dilate)), dims=v.dims)


def occupancy(b: BinaryVolume) -> float:
    """Fraction of voxels flagged (volume.py:322-324)."""
    nx, ny, nz = b.dims
    return float(b.count_nonzero()) / (nx * ny * nz)


# -- raw I/O and generators (fixtures/harness) -----------------------------

def load_raw(path, meta: dict | None = None) -> Volume:
    """A .raw scalar volume (volume.py:165-194): x-fastest on disk.  8-bit files go straight to
    device u8 bins (the field f32(u/255) is implied, no float32 host copy); 16-bit files are
    normalised on the device in float64 and narrowed to float32 like the reference."""
    from pathlib import Path as _P

    path = _P(path)
    if meta is None:
        meta = json.loads(path.with_suffix(path.suffix + ".json").read_text())
    dims = tuple(int(d) for d in meta["dims"])
    bits = int(meta.get("bits", meta.get("bits_per_voxel", 8)))
    endian = meta.get("endian", meta.get("endianness", "little"))
    if bits == 8:
        dtype = np.dtype(np.uint8)
    elif bits == 16:
        dtype = np.dtype(np.uint16).newbyteorder("<" if endian == "little" else ">")
    else:
        raise UnsupportedFormatError(f"unsupported bit depth {bits}")
    raw = path.read_bytes()
    expected = dims[0] * dims[1] * dims[2] * dtype.itemsize
    if len(raw) != expected:
        raise VolumeFormatError(
            f"{path}: file is {len(raw)} bytes, dims {dims} at {bits} bit need {expected}")
    dev = _lib.device()
    flat = np.frombuffer(raw, dtype=dtype)
    if bits == 8:
        t = torch.from_numpy(flat.copy()).to(dev)
        # on disk x fastest: (nz, ny, nx) C-order == (nx, ny, nz) F-order -> permute on device
        vol = t.reshape(dims[2], dims[1], dims[0]).permute(2, 1, 0).contiguous()
        return Volume.from_u8(vol, name=path.stem)
    t = torch.from_numpy(flat.astype(np.int32)).to(dev)
    f64 = t.reshape(dims[2], dims[1], dims[0]).permute(2, 1, 0).double() / float(2 ** bits - 1)
    return Volume(f64.float().contiguous(), name=path.stem)


def save_raw(v: Volume, path, bits: int = 8) -> None:
    """Write .raw + JSON sidecar, x fastest, rint(v * peak) (volume.py:197-206)."""
    from pathlib import Path as _P

    if bits not in (8, 16):
        raise UnsupportedFormatError(f"unsupported bit depth {bits}")
    path = _P(path)
    if bits == 8 and v.field is None:
        q = v.bins  # rint(f32(u/255) * 255) == u
    else:
        src = v.field if v.field is not None else torch.from_numpy(U8_FIELD).to(
            v.bins.device)[v.bins.long()]
        q = torch.round(src.double() * float(2 ** bits - 1))
        q = q.to(torch.uint8) if bits == 8 else q.to(torch.int32)
    arr = q.permute(2, 1, 0).contiguous().cpu().numpy()
    arr = arr.astype(np.uint8 if bits == 8 else "<u2")
    path.write_bytes(arr.tobytes())
    path.with_suffix(path.suffix + ".json").write_text(
        json.dumps({"dims": list(v.dims), "bits": bits, "endian": "little"}))


def gen_menger(level: int) -> Volume:
    """Menger sponge of side 3^level, values 0/1 (volume.py:209-227), built on the device."""
    if level < 0 or level > 6:
        raise ValueError("level must be in [0, 6]")
    dev = _lib.device()
    n = 3 ** level
    c = torch.arange(n, device=dev)
    solid = torch.ones((n, n, n), dtype=torch.bool, device=dev)
    for d in range(level):
        digit = (c // 3 ** d) % 3 == 1
        x, y, z = digit[:, None, None], digit[None, :, None], digit[None, None, :]
        solid &= ~((x & y) | (x & z) | (y & z))
    return Volume.from_u8(solid.to(torch.uint8) * 255, name=f"menger{level}")


def gen_shell(dims, center=None, radius: float = 0.0, thickness: float = 1.0) -> Volume:
    """Spherical shell |(|p - c| - r)| <= t/2 at voxel centres (volume.py:230-248)."""
    if thickness <= 0:
        raise ValueError("thickness must be positive")
    dims = tuple(int(d) for d in dims)
    if center is None:
        center = tuple(d / 2.0 for d in dims)
    dev = _lib.device()
    ax = [torch.arange(d, device=dev, dtype=torch.float64) + 0.5 - c for d, c in zip(dims, center)]
    dist = torch.sqrt(ax[0][:, None, None] ** 2 + ax[1][None, :, None] ** 2 +
                      ax[2][None, None, :] ** 2)
    solid = torch.abs(dist - radius) <= thickness / 2.0
    return Volume.from_u8(solid.to(torch.uint8) * 255, name="shell")


def gen_blobs(dims, n: int, seed: int, sigma: float = 1.5, centers=None) -> Volume:
    """Sum of n Gaussian splats, clamped to [0, 1] (volume.py:251-286), accumulated on the
    device in float64 (summation order differs from numpy's, so the float32 field can differ
    in the last ulp; synth.gen_blobs_u8 gives the 8-bit benchmark volumes)."""
    if n < 1:
        raise ValueError("need at least one blob")
    from .synth import blob_field

    return Volume(blob_field(dims, n, seed, sigma, centers), name="blobs")
