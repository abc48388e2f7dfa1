"""ctypes front-end of the CPU oracle (oracle/vs_oracle.c).

TEST INFRASTRUCTURE ONLY.  This module is the parity checker: tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / ``--impl reference`` leg may import it; the product package
``paper_1912_09596_b200`` never does.  Each wrapper names the reference function it restates
(paths relative to /root/reference/pkg/src/voxelskip/).  The restatement is pinned against
golden vectors produced by the unmodified reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

i64 = C.c_int64
P = C.c_void_p


def build() -> Path:
    """Compile liboracle.so in place (gcc, no FMA contraction)."""
    so = _HERE / "liboracle.so"
    src = _HERE / "vs_oracle.c"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        _LIB = C.CDLL(str(build()))
        L = _LIB
        L.or_classify.restype = i64
        L.or_classify.argtypes = [P, C.c_int, i64, i64, i64, P, C.c_int, P]
        L.or_morton_encode.restype = C.c_uint32
        L.or_morton_encode.argtypes = [i64, i64, i64]
        L.or_flag_bricks.restype = i64
        L.or_flag_bricks.argtypes = [P, i64, i64, i64, i64, P, P, i64]
        L.or_build_lbvh.restype = i64
        L.or_build_lbvh.argtypes = [P, P, i64, i64, i64, i64, i64, P, P, P, P, P, P]
        L.or_svt_build.restype = None
        L.or_svt_build.argtypes = [P, i64, i64, i64, i64, P]
        L.or_box_count.restype = i64
        L.or_box_count.argtypes = [P, i64, i64, i64, i64, P, P]
        L.or_shrink_svt.restype = C.c_int
        L.or_shrink_svt.argtypes = [P, i64, i64, i64, i64, P, P, P, P]
        L.or_tight_box.restype = C.c_int
        L.or_tight_box.argtypes = [P, i64, i64, i64, P, P, P, P]
        L.or_macro_grid.restype = None
        L.or_macro_grid.argtypes = [P, i64, i64, i64, i64, P]
        L.or_cell_boxes.restype = None
        L.or_cell_boxes.argtypes = [P, i64, i64, i64, i64, P, P, P, P, P]
        L.or_snapped_positions.restype = C.c_int
        L.or_snapped_positions.argtypes = [i64, i64, i64, i64, P]
        L.or_kd_build.restype = P
        L.or_kd_build.argtypes = [P, i64, i64, i64, C.c_int, i64, C.c_int, i64, i64]
        L.or_kd_count.restype = i64
        L.or_kd_count.argtypes = [P]
        L.or_kd_root.restype = i64
        L.or_kd_root.argtypes = [P]
        L.or_kd_copy.restype = None
        L.or_kd_copy.argtypes = [P, P, P, P, P, P, P]
        L.or_kd_free.restype = None
        L.or_kd_free.argtypes = [P]
        L.or_render.restype = None
        L.or_render.argtypes = [C.c_int, P, C.c_int, i64, i64, i64, P, P, i64, i64, i64, i64,
                                P, P, P, P, P, P, i64, i64, P, P, i64, i64, i64, i64,
                                C.c_double, C.c_int, P, P, C.c_int]
        L.or_traverse.restype = i64
        L.or_traverse.argtypes = [C.c_int, i64, i64, i64, P, i64, i64, i64, i64, P, P, P, P, P,
                                  P, i64, i64, P, P, P, i64]
        L.or_integrate.restype = None
        L.or_integrate.argtypes = [P, P, P, i64, P, C.c_int, i64, i64, i64, P, C.c_double,
                                   C.c_int, P, P]
        L.or_set_threads.restype = None
        L.or_set_threads.argtypes = [C.c_int]
        L.or_corr_table.restype = None
        L.or_corr_table.argtypes = [P, C.c_double, P]
    return _LIB


def set_threads(n: int) -> None:
    """Host threads for classification / dilation / brick votes (0 = all cores).  Results
    never depend on it (independent x slabs)."""
    lib().or_set_threads(int(n))


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _field(data: np.ndarray):
    """(contiguous array, is_f32).  uint8 volumes stand for f32(u/255) (volume.py:265)."""
    if data.dtype == np.uint8:
        return np.ascontiguousarray(data), 0
    return np.ascontiguousarray(data, dtype=np.float32), 1


def _lut(lut) -> np.ndarray:
    lut = np.ascontiguousarray(lut, dtype=np.float32)
    assert lut.shape == (256, 4)
    return lut


# -- classification (volume.py:231-234, 361-396) -----------------------------------------


def classify(data: np.ndarray, lut, dilate: bool = False):
    """-> (bool flags [x,y,z], count of non-dilated visible voxels)."""
    f, is_f32 = _field(data)
    out = np.zeros(f.shape, dtype=np.uint8)
    cnt = lib().or_classify(_p(f), is_f32, *f.shape, _p(_lut(lut)), int(dilate), _p(out))
    return out.view(bool), int(cnt)


def quantize_u8_identity() -> bool:
    """quantize_scalar(f32(u/255)) == u for every u8 (the device skips quantisation)."""
    tab = (np.arange(256, dtype=np.float64) / 255.0).astype(np.float32)
    q = np.clip(np.floor(tab.astype(np.float64) * 255.0 + 0.5), 0, 255).astype(np.int64)
    return bool(np.array_equal(q, np.arange(256)))


# -- Morton / bricks / LBVH (lbvh.py:25-264) ---------------------------------------------


def morton_encode(x: int, y: int, z: int) -> int:
    return int(lib().or_morton_encode(int(x), int(y), int(z)))


def flag_bricks(bits: np.ndarray, bs: int = 8):
    """-> (coords (n,3) int32 in C scan order, codes (n,) uint32)."""
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    nb = [-(-d // bs) for d in b.shape]
    cap = int(np.prod(nb))
    coords = np.zeros((cap, 3), dtype=np.int32)
    codes = np.zeros(cap, dtype=np.uint32)
    n = lib().or_flag_bricks(_p(b), *b.shape, bs, _p(coords), _p(codes), cap)
    assert n >= 0
    return coords[:n].copy(), codes[:n].copy()


def build_lbvh(coords: np.ndarray, codes: np.ndarray, bs: int, dims) -> dict:
    n = len(coords)
    m = max(2 * n - 1, 0)
    out = {
        "lo": np.zeros((m, 3), np.int32), "hi": np.zeros((m, 3), np.int32),
        "left": np.zeros(m, np.int32), "right": np.zeros(m, np.int32),
        "leaf_brick": np.zeros(m, np.int32), "brick_coords": np.zeros((n, 3), np.int32),
    }
    c = np.ascontiguousarray(coords, dtype=np.int32)
    k = np.ascontiguousarray(codes, dtype=np.uint32)
    h = lib().or_build_lbvh(_p(c), _p(k), n, bs, *dims, _p(out["lo"]), _p(out["hi"]),
                            _p(out["left"]), _p(out["right"]), _p(out["leaf_brick"]),
                            _p(out["brick_coords"]))
    out["root"] = 0 if n else -1
    out["height"] = int(h)
    out["node_count"] = m
    return out


# -- SVT / grid / cells (svt.py:40-195, kdtree.py:285-350) --------------------------------


def svt_build(bits: np.ndarray, bs: int = 32) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    nb = [-(-d // bs) for d in b.shape]
    t = np.zeros((*nb, bs + 1, bs + 1, bs + 1), dtype=np.uint32)
    lib().or_svt_build(_p(b), *b.shape, bs, _p(t))
    return t


def box_count(tables: np.ndarray, dims, bs: int, lo, hi) -> int:
    l = np.asarray(lo, np.int64); h = np.asarray(hi, np.int64)
    return int(lib().or_box_count(_p(np.ascontiguousarray(tables)), *dims, bs, _p(l), _p(h)))


def shrink_svt(tables: np.ndarray, dims, bs: int, lo, hi):
    l = np.asarray(lo, np.int64); h = np.asarray(hi, np.int64)
    ol = np.zeros(3, np.int64); oh = np.zeros(3, np.int64)
    ok = lib().or_shrink_svt(_p(np.ascontiguousarray(tables)), *dims, bs, _p(l), _p(h), _p(ol), _p(oh))
    return (tuple(int(v) for v in ol), tuple(int(v) for v in oh)) if ok else None


def tight_box(bits: np.ndarray, lo, hi):
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    l = np.asarray(lo, np.int64); h = np.asarray(hi, np.int64)
    ol = np.zeros(3, np.int64); oh = np.zeros(3, np.int64)
    ok = lib().or_tight_box(_p(b), *b.shape, _p(l), _p(h), _p(ol), _p(oh))
    return (tuple(int(v) for v in ol), tuple(int(v) for v in oh)) if ok else None


def macro_grid(bits: np.ndarray, cs: int) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    nc = [-(-d // cs) for d in b.shape]
    occ = np.zeros(nc, dtype=np.uint8)
    lib().or_macro_grid(_p(b), *b.shape, cs, _p(occ))
    return occ.view(bool)


def cell_boxes(bits: np.ndarray, cs: int = 8) -> dict:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    nc = [-(-d // cs) for d in b.shape]
    ncell = int(np.prod(nc))
    out = {"codes": np.zeros(ncell, np.uint32), "coords": np.zeros((ncell, 3), np.int32),
           "lo": np.zeros((ncell, 3), np.int32), "hi": np.zeros((ncell, 3), np.int32),
           "occupied": np.zeros(ncell, np.uint8)}
    lib().or_cell_boxes(_p(b), *b.shape, cs, _p(out["codes"]), _p(out["coords"]),
                        _p(out["lo"]), _p(out["hi"]), _p(out["occupied"]))
    out["occupied"] = out["occupied"].view(bool)
    return out


def snapped_positions(lo: int, hi: int, bins: int, cs: int) -> list[int]:
    buf = np.zeros(64, np.int64)
    n = lib().or_snapped_positions(lo, hi, bins, cs, _p(buf))
    return [int(v) for v in buf[:n]]


# -- k-d trees (kdtree.py:387-498) -------------------------------------------------------


def kd_build(bits: np.ndarray, mode: str = "shallow", max_leaf_size=None, builder: str = "sweep",
             bins: int = 4, cell_size: int = 8) -> dict:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    L = lib()
    r = L.or_kd_build(_p(b), *b.shape, int(mode == "deep"),
                      -1 if max_leaf_size is None else int(max_leaf_size),
                      int(builder == "binned"), int(bins), int(cell_size))
    try:
        n = L.or_kd_count(r)
        out = {"lo": np.zeros((n, 3), np.int32), "hi": np.zeros((n, 3), np.int32),
               "axis": np.zeros(n, np.int8), "plane": np.zeros(n, np.int32),
               "left": np.zeros(n, np.int32), "right": np.zeros(n, np.int32)}
        L.or_kd_copy(r, _p(out["lo"]), _p(out["hi"]), _p(out["axis"]), _p(out["plane"]),
                     _p(out["left"]), _p(out["right"]))
        out["root"] = int(L.or_kd_root(r))
    finally:
        L.or_kd_free(r)
    out["node_count"] = n
    out["height"] = kd_height(out)
    return out


def kd_height(t: dict) -> int:
    """kdtree.py:115-127."""
    if len(t["axis"]) == 0:
        return 0
    best, stack = 0, [(t["root"], 1)]
    left, right = t["left"], t["right"]
    while stack:
        i, d = stack.pop()
        best = max(best, d)
        for c in (int(left[i]), int(right[i])):
            if c >= 0:
                stack.append((c, d + 1))
    return best


# -- renderer (render.py:93-149, 196-1015) ------------------------------------------------


def _normalize(v):
    return v / float(np.linalg.norm(v))


def camera_vectors(cam) -> tuple[np.ndarray, np.ndarray]:
    """(eye, up, right, scale) packed as 10 doubles + direction, computed with the same numpy
    operations as Camera.ray_origins (render.py:134-149)."""
    d = np.asarray(cam.direction)
    up = np.asarray(cam.up)
    right = _normalize(np.cross(d, up))
    up = _normalize(np.cross(right, d))
    scale = cam.extent / cam.width
    packed = np.concatenate([np.asarray(cam.eye, np.float64), up, right, [scale]]).astype(np.float64)
    return packed, np.asarray(cam.direction, dtype=np.float64)


def stack_cap(height: int) -> int:
    return max(2 * height + 8, 64)  # render.py:792-793


_KIND = {"naive": 0, "grid": 1, "lbvh": 2, "kd": 3, "hybrid": 4}


def _index_args(kind: str, index: dict | None, dims):
    """index dict keys: grid -> occupied, cell_size; lbvh/kd -> tree arrays; hybrid -> both."""
    z32 = np.zeros((1, 3), np.int32)
    occ = np.zeros(1, np.uint8)
    nc = (1, 1, 1)
    cs = 1
    lo = hi = z32
    left = right = plane = np.zeros(1, np.int32)
    axis = np.zeros(1, np.int8)
    root, height = -1, 0
    if kind in ("grid", "hybrid"):
        occ = np.ascontiguousarray(index["occupied"], dtype=np.uint8)
        nc = occ.shape
        cs = int(index["cell_size"])
    if kind in ("lbvh", "kd", "hybrid"):
        t = index["tree"] if kind == "hybrid" else index
        if len(t["left"]):
            lo = np.ascontiguousarray(t["lo"], np.int32)
            hi = np.ascontiguousarray(t["hi"], np.int32)
            left = np.ascontiguousarray(t["left"], np.int32)
            right = np.ascontiguousarray(t["right"], np.int32)
            if kind != "lbvh":
                axis = np.ascontiguousarray(t["axis"], np.int8)
                plane = np.ascontiguousarray(t["plane"], np.int32)
            root = int(t["root"])
        height = int(t["height"])
    keep = (occ, lo, hi, left, right, axis, plane)
    args = [_p(occ), nc[0], nc[1], nc[2], cs, _p(lo), _p(hi), _p(left), _p(right), _p(axis),
            _p(plane), root, stack_cap(height)]
    return args, keep


def render(kind: str, data: np.ndarray, lut, index: dict | None, cam, dt: float = 0.5,
           nearest: bool = False, rows=None, nthreads: int | None = None):
    """-> (float64 rgba (rows,w,4), int64 samples (rows,w)) for image rows [r0, r1)."""
    f, is_f32 = _field(data)
    lut = _lut(lut)
    packed, direction = camera_vectors(cam)
    w, h = cam.width, cam.height
    r0, r1 = (0, h) if rows is None else rows
    rgba = np.zeros(((r1 - r0) * w, 4), np.float64)
    samples = np.zeros((r1 - r0) * w, np.int64)
    args, keep = _index_args(kind, index, f.shape)
    lib().or_render(_KIND[kind], _p(f), is_f32, *f.shape, _p(lut), *args, _p(packed),
                    _p(direction), w, h, r0, r1, float(dt), int(nearest), _p(rgba), _p(samples),
                    int(nthreads or os.cpu_count() or 1))
    del keep
    return rgba.reshape(r1 - r0, w, 4), samples.reshape(r1 - r0, w)


def quantize_rgba(rgba: np.ndarray) -> np.ndarray:
    """render.py:904."""
    return np.clip(np.floor(rgba * 255.0 + 0.5), 0, 255).astype(np.uint8)


def traverse(kind: str, index: dict | None, dims, origin, direction) -> np.ndarray:
    o = np.asarray(origin, np.float64); d = np.asarray(direction, np.float64)
    args, keep = _index_args(kind, index, dims)
    cap = 4096
    out = np.zeros((cap, 2), np.float64)
    m = lib().or_traverse(_KIND[kind], *dims, *args, _p(o), _p(d), _p(out), cap)
    assert m <= cap
    del keep
    return out[:m].copy()


def integrate(origin, direction, segments: np.ndarray, data: np.ndarray, lut, dt: float = 0.5,
              nearest: bool = False):
    f, is_f32 = _field(data)
    o = np.asarray(origin, np.float64); d = np.asarray(direction, np.float64)
    s = np.ascontiguousarray(np.asarray(segments, np.float64).reshape(-1, 2))
    rgba = np.zeros(4, np.float64)
    samples = np.zeros(1, np.int64)
    lib().or_integrate(_p(o), _p(d), _p(s), len(s), _p(f), is_f32, *f.shape, _p(_lut(lut)),
                       float(dt), int(nearest), _p(rgba), _p(samples))
    return rgba, int(samples[0])


def corr_table(lut, dt: float) -> np.ndarray:
    out = np.zeros(256, np.float64)
    lib().or_corr_table(_p(_lut(lut)), float(dt), _p(out))
    return out


def math_pow_corr(lut, dt: float) -> np.ndarray:
    """Same table with Python's math.pow (== numba's ** on glibc)."""
    lut = _lut(lut)
    return np.array([1.0 - math.pow(1.0 - float(a), dt) for a in lut[:, 3]], np.float64)


def render_multi(kind: str, fields, luts, index: dict | None, cam, dt: float = 0.5, rows=None,
                 nthreads: int | None = None):
    """Multi-channel frame rows [r0, r1) (or_render_multi_rows): u8 channels, one LUT each."""
    L = lib()
    if not hasattr(L, "_multi_bound"):
        L.or_render_multi_rows.restype = None
        L.or_render_multi_rows.argtypes = [C.c_int, P, C.c_int, i64, i64, i64, P, P, i64, i64,
                                           i64, i64, P, P, P, P, P, P, i64, i64, P, P, i64, i64,
                                           i64, i64, C.c_double, P, P, C.c_int]
        L._multi_bound = True
    fs = [np.ascontiguousarray(f, dtype=np.uint8) for f in fields]
    ls = [_lut(l) for l in luts]
    fp = (C.c_void_p * len(fs))(*[f.ctypes.data for f in fs])
    lp = (C.c_void_p * len(ls))(*[l.ctypes.data for l in ls])
    packed, direction = camera_vectors(cam)
    w, h = cam.width, cam.height
    r0, r1 = (0, h) if rows is None else rows
    rgba = np.zeros(((r1 - r0) * w, 4), np.float64)
    samples = np.zeros((r1 - r0) * w, np.int64)
    args, keep = _index_args(kind, index, fs[0].shape)
    L.or_render_multi_rows(_KIND[kind], C.cast(fp, C.c_void_p), len(fs), *fs[0].shape,
                           C.cast(lp, C.c_void_p), *args, _p(packed), _p(direction), w, h, r0, r1,
                           float(dt), _p(rgba), _p(samples), int(nthreads or os.cpu_count() or 1))
    del keep
    return rgba.reshape(r1 - r0, w, 4), samples.reshape(r1 - r0, w)
