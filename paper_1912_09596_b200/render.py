"""Orthographic DVR ray marcher on the B200, drop-in for voxelskip.render
(/root/reference/pkg/src/voxelskip/render.py).

render_frame(v, tf, index, cam, dt, interp) launches one k_render (csrc/render.cu): every
pixel's ray traverses the index (naive / grid DDA / LBVH / k-d / hybrid) and its intervals
are integrated on the reference's sampling lattice as they are emitted, in IEEE double with
the reference's exact operation order, so pixels and sample counts equal the reference's.
The single-ray API (traverse_*, integrate, sample_count_of) runs the same device code on
one-ray batches.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream
from .bench import index_kind
from .hybrid import HybridGrid
from .kdtree import KdTree
from .lbvh import Lbvh
from .svt import MacroGrid
from .volume import TransferFunction, Volume

DEFAULT_DT = 0.5
KIND_ID = {"naive": 0, "grid": 1, "lbvh": 2, "kd": 3, "hybrid": 4}
RF_OVERFLOW, RF_ORDER = 1, 2

# render.py:41 -- what render_frame / index_kind accept as an index
SpatialIndex = None | MacroGrid | Lbvh | KdTree | HybridGrid


def _normalize(v: np.ndarray) -> np.ndarray:
    n = float(np.linalg.norm(v))
    if n == 0.0:
        raise ValueError("zero-length vector")
    return v / n


@dataclass(frozen=True)
class Camera:
    """Orthographic frame (render.py:67-149): rays start on the eye plane, share a direction;
    ``extent`` is the world width of the image, pixels are square."""

    eye: tuple
    direction: tuple
    up: tuple
    extent: float
    width: int
    height: int

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64)
        u = np.asarray(self.up, dtype=np.float64)
        if abs(np.linalg.norm(d) - 1.0) > 1e-6 or abs(np.linalg.norm(u) - 1.0) > 1e-6:
            raise ValueError("direction and up must be unit vectors")
        if np.linalg.norm(np.cross(d, u)) < 1e-6:
            raise ValueError("direction and up are collinear")
        if self.extent <= 0 or self.width < 1 or self.height < 1:
            raise ValueError("bad viewport")

    @classmethod
    def orbit(cls, dims, azimuth_deg: float, elevation_deg: float = 0.0, zoom: float = 1.0,
              width: int = 512, height: int | None = None) -> "Camera":
        """On the bounding sphere, orbiting the vertical (y) axis, looking at the centre."""
        if zoom <= 0:
            raise ValueError("zoom must be positive")
        center = np.asarray(dims, dtype=np.float64) * 0.5
        diameter = float(np.linalg.norm(np.asarray(dims, dtype=np.float64)))
        az = math.radians(azimuth_deg)
        el = math.radians(max(-89.9, min(89.9, elevation_deg)))
        u = np.array([math.cos(el) * math.sin(az), math.sin(el), math.cos(el) * math.cos(az)])
        eye = center + diameter * u
        d = _normalize(center - eye)
        right = np.cross(d, np.array([0.0, 1.0, 0.0]))
        if np.linalg.norm(right) < 1e-9:
            right = np.array([1.0, 0.0, 0.0])
        right = _normalize(right)
        up = _normalize(np.cross(right, d))
        return cls(eye=tuple(eye), direction=tuple(d), up=tuple(up), extent=diameter / zoom,
                   width=width, height=height if height is not None else width)

    def frame_vectors(self):
        """(eye, up, right, scale) exactly as ray_origins derives them."""
        d = np.asarray(self.direction)
        up = np.asarray(self.up)
        right = _normalize(np.cross(d, up))
        up = _normalize(np.cross(right, d))
        return np.asarray(self.eye, dtype=np.float64), up, right, self.extent / self.width

    def ray_origins(self) -> np.ndarray:
        """(h*w, 3) origins, row-major, top row first (host helper)."""
        eye, up, right, scale = self.frame_vectors()
        xs = (np.arange(self.width) + 0.5 - self.width / 2.0) * scale
        ys = (self.height / 2.0 - np.arange(self.height) - 0.5) * scale
        o = eye[None, None, :] + ys[:, None, None] * up[None, None, :] + \
            xs[None, :, None] * right[None, None, :]
        return np.ascontiguousarray(o.reshape(-1, 3), dtype=np.float64)


@dataclass(frozen=True)
class Ray:
    origin: tuple
    direction: tuple


@dataclass
class RaySegmentList:
    """Sorted disjoint [t0, t1) intervals to integrate along one ray."""

    t: np.ndarray

    def __post_init__(self):
        self.t = np.asarray(self.t, dtype=np.float64).reshape(-1, 2)

    @property
    def count(self) -> int:
        return int(self.t.shape[0])

    def as_pairs(self):
        return [(float(a), float(b)) for a, b in self.t]


@dataclass
class Frame:
    """Premultiplied RGBA8 image plus the number of field samples taken (render.py:175-190)."""

    width: int
    height: int
    pixels: np.ndarray
    sample_count: int

    def to_raw(self) -> bytes:
        return self.pixels.tobytes()

    def to_png(self, path) -> None:
        from PIL import Image

        Image.fromarray(self.pixels, mode="RGBA").save(path)


# -- C structs (include/vsb200.h) --------------------------------------------------------------
class VolumeDesc(C.Structure):
    _fields_ = [("bins", C.c_void_p), ("field", C.c_void_p), ("nx", C.c_int), ("ny", C.c_int),
                ("nz", C.c_int), ("pad", C.c_int), ("quads", C.c_void_p)]


class IndexDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("root", C.c_int), ("occ", C.c_void_p), ("ncx", C.c_int),
                ("ncy", C.c_int), ("ncz", C.c_int), ("cs", C.c_int), ("lo", C.c_void_p),
                ("hi", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p),
                ("plane", C.c_void_p), ("axis", C.c_void_p), ("lbvh_info", C.c_void_p),
                ("brick_bits", C.c_void_p), ("nbx", C.c_int), ("nby", C.c_int), ("nbz", C.c_int),
                ("bs", C.c_int)]


class CameraDesc(C.Structure):
    _fields_ = [("eye", C.c_double * 3), ("up", C.c_double * 3), ("right", C.c_double * 3),
                ("dir", C.c_double * 3), ("scale", C.c_double), ("width", C.c_int),
                ("height", C.c_int)]


class RowsDesc(C.Structure):
    _fields_ = [("nrows", C.c_int), ("stripe", C.c_int), ("nparts", C.c_int), ("part", C.c_int)]


# vs_render_opts code-path bits (include/vsb200.h); every combination gives the same frame
RO_U8_TABLE, RO_FP64_BINS, RO_GENERIC_TRAVERSAL, RO_BRICK_NO_RUNS = 1, 2, 4, 16
RO_DEFAULT = RO_U8_TABLE


class RenderOpts(C.Structure):
    """vs_render_opts: every renderer setting travels with the call (no library state)."""

    _fields_ = [("ert_eps", C.c_double), ("flags", C.c_int), ("trav_steps", C.c_int),
                ("sample_steps", C.c_int), ("reserved", C.c_int)]


def render_opts(ert_eps: float = 0.0, flags: int = RO_DEFAULT, trav_steps: int = 1,
                sample_steps: int = 1) -> RenderOpts:
    return RenderOpts(float(ert_eps), int(flags), int(trav_steps), int(sample_steps), 0)


def volume_desc(v: Volume, quads: bool = True) -> VolumeDesc:
    nx, ny, nz = v.dims
    q = v.quads() if (quads and v.field is None) else None
    return VolumeDesc(ptr(v.bins), ptr(v.field), nx, ny, nz, 0, ptr(q))


def camera_desc(cam: Camera) -> CameraDesc:
    eye, up, right, scale = cam.frame_vectors()
    d = np.asarray(cam.direction, dtype=np.float64)
    c = CameraDesc()
    for k in range(3):
        c.eye[k], c.up[k], c.right[k], c.dir[k] = float(eye[k]), float(up[k]), float(right[k]), \
            float(d[k])
    c.scale, c.width, c.height = float(scale), int(cam.width), int(cam.height)
    return c


_EMPTY = {}


def _placeholder() -> int:
    """A valid device address for the arrays of an empty tree (root -1: never read)."""
    dev = _lib.device()
    if dev.index not in _EMPTY:
        _EMPTY[dev.index] = torch.zeros(16, dtype=torch.int32, device=dev)
    return ptr(_EMPTY[dev.index])


def index_desc(index, use_brick_dda: bool = True) -> IndexDesc:
    """Descriptor + the tensors it points at (keep them alive for the launch)."""
    kind = index_kind(index)
    d = IndexDesc()
    d.kind = KIND_ID[kind]
    d.root = -1
    if kind in ("grid", "hybrid"):
        g: MacroGrid = index if kind == "grid" else index.grid
        d.occ = ptr(g.occupied_dev)
        d.ncx, d.ncy, d.ncz = g.cells_dims
        d.cs = g.cell_size
    if kind == "lbvh":
        t: Lbvh = index
        d.lo, d.hi = ptr(t.dev["lo"]), ptr(t.dev["hi"])
        d.left, d.right = ptr(t.dev["left"]), ptr(t.dev["right"])
        d.lbvh_info = ptr(t.info)
        if use_brick_dda:
            d.brick_bits = ptr(t.brick_grid())
            d.nbx, d.nby, d.nbz = t.brick_grid_dims()
            d.bs = t.brick_size
    if kind in ("kd", "hybrid"):
        t = index if kind == "kd" else index.tree
        dv = t.device_arrays()
        d.lo, d.hi, d.left, d.right = ptr(dv["lo"]), ptr(dv["hi"]), ptr(dv["left"]), \
            ptr(dv["right"])
        d.plane, d.axis = ptr(dv["plane"]), ptr(dv["axis"])
        d.root = int(t.root)
    if kind in ("lbvh", "kd", "hybrid"):
        for f in ("lo", "hi", "left", "right", "plane", "axis"):
            if not getattr(d, f):
                setattr(d, f, _placeholder())  # empty tree: root -1 / 0 bricks
    return d


def tf_device(tf: TransferFunction, dt: float):
    """(lut float32 (256,4), corr float64 (256,)) on the device for (tf, dt).  corr uses
    Python's math.pow, which is the C library pow numba's ** calls (render.py:752)."""
    dev = _lib.device()
    key = ("render", dev.index, float(dt))
    cache = tf._dev
    if key not in cache:
        corr = np.array([1.0 - math.pow(1.0 - float(a), float(dt)) for a in tf.lut[:, 3]],
                        dtype=np.float64)
        cache[key] = (_lib.upload(tf.lut), _lib.upload(corr))  # stream-ordered, no host wait
    return cache[key]


def _check_flags(flags: torch.Tensor):
    _check_flag_bits(int(flags.item()))


def _check_flag_bits(f: int):
    if f & RF_OVERFLOW:
        raise RuntimeError("traversal stack overflow (tree deeper than the device stack)")
    if f & RF_ORDER:
        raise RuntimeError("non-monotone interval emission (streaming merge would differ)")


SEG_CAP = 32  # lattice ranges per ray kept between the traversal and integration kernels


class RenderTarget:
    """Device output buffers for render_rows (reused across frames), plus the two-phase
    segment workspace (``seg_cap`` = 0 selects the fused single-kernel path)."""

    def __init__(self, width: int, nrows: int, want_rgba64=False, want_samples=False,
                 seg_cap: int = SEG_CAP):
        dev = _lib.device()
        self.seg_cap = int(seg_cap)
        wsb = _lib.query("vs_render_workspace", width * nrows, self.seg_cap)
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
        self.rgba8 = torch.empty((nrows, width, 4), dtype=torch.uint8, device=dev)
        self.rgba64 = torch.empty((nrows, width, 4), dtype=torch.float64, device=dev) \
            if want_rgba64 else None
        self.samples = torch.empty((nrows, width), dtype=torch.int32, device=dev) \
            if want_samples else None
        self.total = torch.zeros(1, dtype=torch.int64, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)


def render_rows(v: Volume, tf: TransferFunction, index, cam: Camera, target: RenderTarget,
                dt: float = DEFAULT_DT, nearest: bool = False, rows: RowsDesc | None = None,
                idx_desc: IndexDesc | None = None, vol_desc: VolumeDesc | None = None,
                cam_desc: CameraDesc | None = None, zero: bool = True, ert_eps: float = 0.0,
                flags: int = RO_DEFAULT, opts: RenderOpts | None = None):
    """Launch the renderer for (a stripe set of) the frame into ``target`` (async).

    ``ert_eps`` > 0 enables early ray termination at accumulated opacity 1 - ert_eps (RGBA
    within ert_eps of the full integral, fewer samples); 0 is the reference's integrator.
    ``flags`` picks code paths (RO_*; identical results).  ``opts`` overrides both."""
    lut, corr = tf_device(tf, dt)
    if zero:
        target.total.zero_()
        target.flags.zero_()
    idx_desc = idx_desc or index_desc(index)
    vol_desc = vol_desc or volume_desc(v)
    cam_desc = cam_desc or camera_desc(cam)
    opts = opts or render_opts(ert_eps, flags)
    call("vs_render", C.addressof(vol_desc), C.addressof(idx_desc), C.addressof(cam_desc),
         ptr(lut), ptr(corr), float(dt), int(nearest),
         None if rows is None else C.addressof(rows), ptr(target.rgba8), ptr(target.rgba64),
         ptr(target.samples), ptr(target.total), ptr(target.flags), ptr(target.ws),
         0 if target.ws is None else target.ws.numel(), target.seg_cap, C.addressof(opts),
         stream())


def render_frame(v: Volume, tf: TransferFunction, index, cam: Camera, dt: float = DEFAULT_DT,
                 interp: str = "trilinear") -> Frame:
    """March every pixel's ray through the index and composite front to back
    (render.py:869-911).  Alpha is accumulated opacity, colours premultiplied."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    if interp not in ("trilinear", "nearest"):
        raise ValueError(f"unknown interpolation: {interp!r}")
    tgt = RenderTarget(cam.width, cam.height)
    render_rows(v, tf, index, cam, tgt, dt=dt, nearest=interp == "nearest")
    _check_flags(tgt.flags)
    return Frame(width=cam.width, height=cam.height, pixels=tgt.rgba8.cpu().numpy(),
                 sample_count=int(tgt.total.item()))


def render_float(v: Volume, tf: TransferFunction, index, cam: Camera, dt: float = DEFAULT_DT,
                 interp: str = "trilinear", ert_eps: float = 0.0, flags: int = RO_DEFAULT,
                 rows: RowsDesc | None = None):
    """(float64 premultiplied RGBA (h,w,4), per-pixel samples (h,w)) -- the float output the
    parity tests compare with the reference's _k_integrate accumulators.  ``rows`` renders a
    row band / stripe set only (shape (rows.nrows, w, ...))."""
    nrows = cam.height if rows is None else rows.nrows
    tgt = RenderTarget(cam.width, nrows, want_rgba64=True, want_samples=True)
    render_rows(v, tf, index, cam, tgt, dt=dt, nearest=interp == "nearest", rows=rows,
                ert_eps=ert_eps, flags=flags)
    _check_flags(tgt.flags)
    return tgt.rgba64.cpu().numpy(), tgt.samples.cpu().numpy().astype(np.int64)


# -- single-ray interface (render.py:917-1015) ---------------------------------------------------

def _dims_of(index, dims=None):
    if dims is not None:
        return tuple(int(d) for d in dims)
    kind = index_kind(index)
    if kind == "hybrid":
        return index.tree.dims
    return index.dims


def _traverse(index, dims, ray: Ray) -> RaySegmentList:
    dev = _lib.device()
    o = torch.tensor([ray.origin], dtype=torch.float64, device=dev)
    d = torch.tensor(ray.direction, dtype=torch.float64, device=dev)
    cap = 4096
    out = torch.empty((1, cap, 2), dtype=torch.float64, device=dev)
    counts = torch.zeros(1, dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    desc = index_desc(index)
    nx, ny, nz = dims
    call("vs_traverse_rays", C.addressof(desc), nx, ny, nz, ptr(o), ptr(d), 1, ptr(out), cap,
         ptr(counts), ptr(flags), stream())
    _check_flags(flags)
    m = int(counts.item())
    if m > cap:
        raise RuntimeError("more than 4096 intervals on one ray")
    return RaySegmentList(t=out[0, :m].cpu().numpy())


def traverse_naive(ray: Ray, dims) -> RaySegmentList:
    return _traverse(None, tuple(dims), ray)


def traverse_grid(ray: Ray, grid: MacroGrid) -> RaySegmentList:
    return _traverse(grid, grid.dims, ray)


def traverse_lbvh(ray: Ray, idx: Lbvh) -> RaySegmentList:
    return _traverse(idx, idx.dims, ray)


def traverse_kd(ray: Ray, idx) -> RaySegmentList:
    return _traverse(idx, idx.dims, ray)


def traverse_hybrid(ray: Ray, idx) -> RaySegmentList:
    return _traverse(idx, idx.tree.dims, ray)


def _integrate(ray: Ray, segments: RaySegmentList, v: Volume, lut, corr, dt, nearest):
    dev = _lib.device()
    o = torch.tensor([ray.origin], dtype=torch.float64, device=dev)
    d = torch.tensor(ray.direction, dtype=torch.float64, device=dev)
    m = segments.count
    segs = torch.zeros((1, max(m, 1), 2), dtype=torch.float64, device=dev)
    if m:
        segs[0, :m] = torch.from_numpy(segments.t).to(dev)
    counts = torch.tensor([m], dtype=torch.int32, device=dev)
    rgba = torch.zeros((1, 4), dtype=torch.float64, device=dev)
    samples = torch.zeros(1, dtype=torch.int64, device=dev)
    vd = volume_desc(v)
    call("vs_integrate_rays", C.addressof(vd), ptr(o), ptr(d), ptr(segs), ptr(counts),
         max(m, 1), 1, ptr(lut), ptr(corr), float(dt), int(nearest), ptr(rgba), ptr(samples),
         stream())
    return rgba[0].cpu().numpy(), int(samples.item())


def integrate(ray: Ray, segments: RaySegmentList, v: Volume, tf: TransferFunction,
              dt: float = DEFAULT_DT, interp: str = "trilinear") -> np.ndarray:
    """Composite one ray over its segments on the lattice anchored at the volume entry."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    lut, corr = tf_device(tf, dt)
    rgba, _ = _integrate(ray, segments, v, lut, corr, dt, interp == "nearest")
    return rgba


def sample_count_of(ray: Ray, segments: RaySegmentList, dims, dt: float = DEFAULT_DT) -> int:
    """Lattice points of the ray inside the segments."""
    dev = _lib.device()
    v = Volume.from_u8(torch.zeros(tuple(int(d) for d in dims), dtype=torch.uint8, device=dev))
    lut = torch.zeros((256, 4), dtype=torch.float32, device=dev)
    corr = torch.zeros(256, dtype=torch.float64, device=dev)
    _, n = _integrate(ray, segments, v, lut, corr, dt, False)
    return n
