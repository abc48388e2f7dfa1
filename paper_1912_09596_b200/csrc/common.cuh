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

// SM count of the current device (a cheap attribute query; no cached global state).
inline int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
    n = 148;
  return n;
}

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

// ---- the renderer's trilinear gather ("quad") volume ---------------------------------------
// One 32-bit word per voxel: its 2x2 (y, z) neighbourhood.  Stored in 4x4x4-voxel tiles (64
// words = two 128-byte lines of 2x4x4 voxels each, tiles in C order, words in C order inside a
// tile), so the 32 samples a warp takes at one lattice index -- a small patch of the plane
// normal to the rays, at any orientation -- touch a few lines instead of one line per (x, y)
// row, and a ray's next samples stay in the same tiles.  VS_QUAD_LINEAR: plain C order.
#ifndef VS_QUAD_LINEAR
#ifndef VS_QT_X
#define VS_QT_X 2  // log2 tile edge along x, y, z
#endif
#ifndef VS_QT_Y
#define VS_QT_Y 2
#endif
#ifndef VS_QT_Z
#define VS_QT_Z 2
#endif
struct QuadGeom {
  static constexpr uint32_t LX = VS_QT_X, LY = VS_QT_Y, LZ = VS_QT_Z, T = 1u << (LX + LY + LZ);
  uint32_t ntz, tsx;  // tiles along z; words per x row of tiles
  __host__ __device__ QuadGeom(int nx, int ny, int nz)
      : ntz(((uint32_t)nz + (1u << LZ) - 1) >> LZ),
        tsx((((uint32_t)ny + (1u << LY) - 1) >> LY) * (((uint32_t)nz + (1u << LZ) - 1) >> LZ) * T) {
    (void)nx;
  }
  __host__ __device__ static int64_t words(int nx, int ny, int nz) {
    return (int64_t)((nx + (1 << LX) - 1) >> LX) * ((ny + (1 << LY) - 1) >> LY) *
           ((nz + (1 << LZ) - 1) >> LZ) * T;
  }
  // word index of voxel (x, y, z): tile part + in-tile part
  __host__ __device__ uint32_t yz(int y, int z) const {
    return (((uint32_t)y >> LY) * ntz + ((uint32_t)z >> LZ)) * T +
           (((uint32_t)y & ((1u << LY) - 1)) << LZ) + ((uint32_t)z & ((1u << LZ) - 1));
  }
  __host__ __device__ uint32_t at(int x, uint32_t yzw) const {
    return ((uint32_t)x >> LX) * tsx + (((uint32_t)x & ((1u << LX) - 1)) << (LY + LZ)) + yzw;
  }
};
#else
struct QuadGeom {
  uint32_t ny, nz;
  __host__ __device__ QuadGeom(int nx, int ny_, int nz_) : ny((uint32_t)ny_), nz((uint32_t)nz_) {
    (void)nx;
  }
  __host__ __device__ static int64_t words(int nx, int ny, int nz) {
    return (int64_t)nx * ny * nz;
  }
  __host__ __device__ uint32_t yz(int y, int z) const { return (uint32_t)y * nz + (uint32_t)z; }
  __host__ __device__ uint32_t at(int x, uint32_t yzw) const { return (uint32_t)x * ny * nz + yzw; }
};
#endif

// Packed bit volume: one 32-bit word per 32 voxels along z; word (x, y, w) at
// (x*ny + y)*nzw + w, bit z & 31.
__host__ __device__ inline int64_t nzw_of(int nz) { return (nz + 31) >> 5; }

#ifdef __CUDACC__
// A trilinear sample's classification bin floor(v*255 + 0.5) (render.py:694-748) from its
// 2x2x2 u8 neighbourhood (quad words w0 = x0 plane, w1 = x1 plane; tb = f32(u/255) table) in
// FP32, when that is provably the bin of the reference's evaluation (f32 first differences, FP64
// lerps), else -1.  Error of v against the reference: < 9.0e-7 (fractions rounded to f32:
// 2^-25; FMA and difference roundings: 2^-25 each on values in [0, 1]; three lerp levels), so
// w = v*255 + 0.5 is within 2.4e-4 (+ its own rounding, 7.6e-6 at 255.5) of the reference's; a
// fractional part of w at least BIN_EDGE from an integer fixes floor(w).  ~0.2% of samples
// fall back to the FP64 evaluation.
constexpr float BIN_EDGE = 1e-3f;
// Byte-domain variant (default): the same test on 255·v evaluated from the raw bytes, so no
// shared-memory table reads (8 LDS per sample) compete with the gathers for L1TEX.  A byte u
// becomes the float 2^23 + u by one PRMT into the mantissa of 2^23 (0x4B0000uu), exact; the
// first differences of those are the exact byte differences, and one FADD of -2^23 (exact)
// unbiases each lerp base.  Error of w' = lerp(bytes) + 0.5 against
// the reference's v*255 + 0.5: table values f32(u/255)*255 vs u <= 1.6e-5, the reference's f32
// difference roundings x255 <= 7.6e-6 per difference, our three FMA levels on values <= 255.5
// at 2^-24 relative (1.6e-5 each) and the f32 fractions (<= 255 * 2^-25 = 7.6e-6 per level):
// < 1.4e-4 in total, well inside BIN_EDGE.
__device__ __forceinline__ float byte_b(uint32_t w, uint32_t sel) {  // 2^23 + byte, exact
  return __int_as_float((int)__byte_perm(w, 0x4B000000u, sel));
}
__device__ __forceinline__ int bin_fast_bytes(uint32_t w0, uint32_t w1, float fx, float fy,
                                              float fz) {
  // biased corners 2^23 + u: their differences are the exact byte differences, and only the
  // four x0 corners need the bias removed
  const float b000 = byte_b(w0, 0x7440), b001 = byte_b(w0, 0x7441);
  const float b010 = byte_b(w0, 0x7442), b011 = byte_b(w0, 0x7443);
  const float b100 = byte_b(w1, 0x7440), b101 = byte_b(w1, 0x7441);
  const float b110 = byte_b(w1, 0x7442), b111 = byte_b(w1, 0x7443);
  const float c00 = __fmaf_rn(__fsub_rn(b100, b000), fx, __fadd_rn(b000, -8388608.0f));
  const float c10 = __fmaf_rn(__fsub_rn(b110, b010), fx, __fadd_rn(b010, -8388608.0f));
  const float c01 = __fmaf_rn(__fsub_rn(b101, b001), fx, __fadd_rn(b001, -8388608.0f));
  const float c11 = __fmaf_rn(__fsub_rn(b111, b011), fx, __fadd_rn(b011, -8388608.0f));
  const float c0 = __fmaf_rn(__fsub_rn(c10, c00), fy, c00);
  const float c1 = __fmaf_rn(__fsub_rn(c11, c01), fy, c01);
  const float w = __fadd_rn(__fmaf_rn(__fsub_rn(c1, c0), fz, c0), 0.5f);
  const float fl = floorf(w), fr = __fsub_rn(w, fl);
  if (fr < BIN_EDGE || fr > 1.0f - BIN_EDGE) return -1;
  const int bi = (int)fl;
  return bi < 0 ? 0 : (bi > 255 ? 255 : bi);
}
// Table variant (f32(u/255) from a shared-memory table; build with VS_BIN_TABLE for A/B).  The
// byte variant is faster in both integrators once their gathers are software-pipelined (the
// table's 8 LDS per channel per sample compete with the gathers for L1TEX).
__device__ __forceinline__ int bin_fast_table(const float* tb, uint32_t w0, uint32_t w1, float fx,
                                              float fy, float fz) {
  const float c000 = tb[w0 & 0xffu], c001 = tb[(w0 >> 8) & 0xffu];
  const float c010 = tb[(w0 >> 16) & 0xffu], c011 = tb[w0 >> 24];
  const float c100 = tb[w1 & 0xffu], c101 = tb[(w1 >> 8) & 0xffu];
  const float c110 = tb[(w1 >> 16) & 0xffu], c111 = tb[w1 >> 24];
  const float c00 = __fmaf_rn(__fsub_rn(c100, c000), fx, c000);
  const float c10 = __fmaf_rn(__fsub_rn(c110, c010), fx, c010);
  const float c01 = __fmaf_rn(__fsub_rn(c101, c001), fx, c001);
  const float c11 = __fmaf_rn(__fsub_rn(c111, c011), fx, c011);
  const float c0 = __fmaf_rn(__fsub_rn(c10, c00), fy, c00);
  const float c1 = __fmaf_rn(__fsub_rn(c11, c01), fy, c01);
  const float v = __fmaf_rn(__fsub_rn(c1, c0), fz, c0);
  const float w = __fmaf_rn(v, 255.0f, 0.5f);
  const float fl = floorf(w), fr = __fsub_rn(w, fl);
  if (fr < BIN_EDGE || fr > 1.0f - BIN_EDGE) return -1;
  const int bi = (int)fl;
  return bi < 0 ? 0 : (bi > 255 ? 255 : bi);
}
#ifndef VS_BIN_TABLE
__device__ __forceinline__ int bin_fast(const float*, uint32_t w0, uint32_t w1, float fx, float fy,
                                        float fz) {
  return bin_fast_bytes(w0, w1, fx, fy, fz);
}
#else
__device__ __forceinline__ int bin_fast(const float* tb, uint32_t w0, uint32_t w1, float fx,
                                        float fy, float fz) {
  return bin_fast_table(tb, w0, w1, fx, fy, fz);
}
#endif
#endif

}  // namespace vs
