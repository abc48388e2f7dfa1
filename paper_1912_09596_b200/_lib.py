"""ctypes binding of libvsb200.so (include/vsb200.h).

The product path has no CPU fallback: if the library is missing or no CUDA device is present,
every device entry point raises.  Status codes follow the header: 0 ok, negative argument
errors, positive cudaError_t; failures raise with the library's thread-local message.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("VSB200_LIB", str(_PKG / "libvsb200.so")))  # override: dev tuning

i32, i64, u64, P, SZ = C.c_int, C.c_int64, C.c_uint64, C.c_void_p, C.c_size_t

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "vs_version": (C.c_char_p, []),
    "vs_last_error": (i32, [C.c_char_p, SZ]),
    "vs_tf_params_from_alpha": (i32, [P, P]),
    "vs_quantize_f32": (i32, [P, i64, P, P]),
    "vs_classify_summary": (i32, [P, i32, i32, i32, P, P, P, P, P]),
    "vs_classify_bits": (i32, [P, i32, i32, i32, P, P, P, P]),
    "vs_classify_dilate_bits": (i32, [P, i32, i32, i32, P, P, P, P]),
    "vs_classify_dilate_bits_bbox": (i32, [P, i32, i32, i32, P, P, P, P, P]),
    "vs_dilate_bits": (i32, [P, i32, i32, i32, P, P]),
    "vs_pack_bits": (i32, [P, i32, i32, i32, P, P]),
    "vs_unpack_bits": (i32, [P, i32, i32, i32, P, P]),
    "vs_count_bits": (i32, [P, i32, i32, i32, P, P]),
    "vs_vote_cells": (i32, [P, i32, i32, i32, i32, P, P]),
    "vs_morton_side": (i32, [i32, i32, i32]),
    "vs_summary_to_bitmap": (i32, [P, i32, i32, i32, i32, i32, P, P, P, P, P]),
    "vs_presence_words": (i64, [i32, i32, i32]),
    "vs_presence_build": (i32, [P, i32, i32, i32, P, P]),
    "vs_presence_build_slab": (i32, [P, i32, i32, i32, i32, i32, P, P]),
    "vs_presence_to_bitmap": (i32, [P, P, i32, i32, i32, i32, i32, P, P, P, P, P]),
    "vs_flags_to_bitmap": (i32, [P, i32, i32, i32, i32, P, P, P]),
    "vs_bricks_workspace": (SZ, [i32, i32, i32]),
    "vs_bricks_from_bitmap": (i32, [P, i32, i32, i32, i32, P, P, P, P, SZ, P]),
    "vs_lbvh_workspace": (SZ, [i32, i64]),
    "vs_lbvh_from_bitmap": (i32, [P, P, i32, i32, i32, i32, i32, i64, P, P, P, P, P, P, P, P,
                                  P, SZ, P]),
    "vs_lbvh_height_workspace": (SZ, [i64]),
    "vs_lbvh_height": (i32, [P, P, P, i64, P, SZ, P]),
    "vs_lbvh_bricks_workspace": (SZ, [i64]),
    "vs_svt_build": (i32, [P, i32, i32, i32, i32, P, P]),
    "vs_box_count": (i32, [P, i32, i32, i32, i32, P, i32, P, P]),
    "vs_tight_box": (i32, [P, i32, i32, i32, P, P, P]),
    "vs_kd_build": (i32, [P, i32, i32, i32, i32, i32, i32, i32, i32, P, P]),
    "vs_kd_build_bbox": (i32, [P, i32, i32, i32, P, i32, i32, i32, i32, i32, P, P]),
    "vs_kd_result_info": (i32, [P, P, P, P]),
    "vs_kd_result_copy": (i32, [P, P, P, P, P, P, P, P]),
    "vs_kd_result_free": (None, [P]),
    "vs_cell_boxes": (i32, [P, i32, i32, i32, i32, P, P, P, P]),
    "vs_kd_best_plane": (i32, [P, i32, i32, i32, P, i32, i32, i32, P, P]),
    "vs_build_quads": (i32, [P, i32, i32, i32, P, P]),
    "vs_quads_words": (i64, [i32, i32, i32]),
    "vs_mquads_words": (i32, [i32]),
    "vs_mquads_size": (i64, [i32, i32, i32, i32]),
    "vs_build_mquads": (i32, [P, i32, i32, i32, i32, P, P]),
    "vs_or_words": (i32, [P, P, i64, P]),
    "vs_render_multi_integrate": (i32, [P, P, C.c_double, P, P, P, i32, P, P, P, P, P, P]),
    "vs_render_segments": (i32, [P, P, P, C.c_double, P, P, P, i32, P, P, P]),
    "vs_lbvh_brick_grid": (i32, [P, P, i64, i32, i32, i32, P, P]),
    "vs_render": (i32, [P, P, P, P, P, C.c_double, i32, P, P, P, P, P, P, P, SZ, i32, P, P]),
    "vs_render_workspace": (SZ, [i64, i32]),
    "vs_traverse_rays": (i32, [P, i32, i32, i32, P, P, i32, P, i32, P, P, P]),
    "vs_integrate_rays": (i32, [P, P, P, P, P, i32, i32, P, P, C.c_double, i32, P, P, P]),
    "vs_lbvh_from_bricks": (i32, [P, P, i64, i32, i32, i32, i32, P, P, P, P, P, P, P, P, SZ,
                                  P]),
}

_lib = None


class VsError(RuntimeError):
    """A libvsb200 call failed (argument error or CUDA error)."""


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise VsError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python -m paper_1912_09596_b200._build)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    buf = C.create_string_buffer(512)
    lib().vs_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def call(name: str, *args) -> int:
    st = getattr(lib(), name)(*args)
    if st != 0:
        raise VsError(f"{name} failed with status {st}: {last_error()}")
    return st


def query(name: str, *args) -> int:
    return int(getattr(lib(), name)(*args))


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise VsError("paper_1912_09596_b200 needs a CUDA device (B200, sm_100a); "
                      "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def upload(arr) -> torch.Tensor:
    """Host array -> device without blocking the host: staged in pinned memory from torch's
    caching host allocator (which keeps the block until the stream-ordered copy has run)."""
    import numpy as np

    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()  # torch.from_numpy wants a writable array (read-only LUTs)
    host = torch.from_numpy(a).pin_memory()
    return host.to(device(), non_blocking=True)


def workspace(nbytes: int) -> torch.Tensor:
    """Scratch from torch's caching allocator (stream-ordered on the current stream)."""
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device())
