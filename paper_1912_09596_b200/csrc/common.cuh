// Shared device helpers and the C-ABI error convention for libvsb200.so.
//
// Status convention (include/vsb200.h): 0 = ok, negative = argument error (VS_E*),
// positive = a cudaError_t.  The message of the last failure on the calling host thread is
// kept in a thread-local buffer and returned by vs_last_error().
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/vsb200.h"

namespace vs {

void set_error(const char* fmt, ...);

inline int fail_arg(const char* what) {
  set_error("invalid argument: %s", what);
  return VS_EINVAL;
}

inline int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

#define VS_TRY(expr)              \
  do {                            \
    int _st = (expr);             \
    if (_st != 0) return _st;     \
  } while (0)

#define VS_CUDA(expr, where)                                         \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) {                                         \
      ::vs::set_error("%s: %s", where, cudaGetErrorString(_e));      \
      return (int)_e;                                                \
    }                                                                \
  } while (0)

inline cudaStream_t S(vs_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Bump allocator over a caller-provided device workspace (CUB two-phase style: a null base
// only measures).
struct Bump {
  char* base;
  size_t off = 0;
  explicit Bump(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

// ---- Morton (lbvh.py:25-66): 10 bits per axis, x -> bit 3i, y -> 3i+1, z -> 3i+2 ----------
__host__ __device__ inline uint32_t spread10(uint32_t v) {
  v &= 0x3FFu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__host__ __device__ inline uint32_t compact10(uint32_t v) {
  v &= 0x09249249u;
  v = (v | (v >> 2)) & 0x030C30C3u;
  v = (v | (v >> 4)) & 0x0300F00Fu;
  v = (v | (v >> 8)) & 0x030000FFu;
  v = (v | (v >> 16)) & 0x000003FFu;
  return v;
}
__host__ __device__ inline uint32_t morton3(uint32_t x, uint32_t y, uint32_t z) {
  return spread10(x) | (spread10(y) << 1) | (spread10(z) << 2);
}

// Packed bit volume: one 32-bit word per 32 voxels along z; word (x, y, w) at
// (x*ny + y)*nzw + w, bit z & 31.
__host__ __device__ inline int64_t nzw_of(int nz) { return (nz + 31) >> 5; }

}  // namespace vs
