// TF classification kernels: the fused brick-summary pass, packed bit volumes, dilation,
// cell votes and the Morton bitmap of non-empty bricks.
//
// Reference semantics (paths relative to /root/reference/pkg/src/voxelskip/):
//   quantize_scalar  volume.py:159-162   floor(v*255+0.5) clipped, float64
//   classify         volume.py:307-319   visible <=> lut[bin, 3] > 0
//   _dilate26        volume.py:289-304   3x3x3 box OR, clipped at the borders
//   occupancy        volume.py:322-324   count_nonzero / size (undilated at the call sites)
//   flag_bricks      lbvh.py:83-102      padded reshape-any per brick, C scan order
//   _macro_from_bits svt.py:161-167      same vote with cell edge cs
//
// The hot kernel is k_brick_summary: one coalesced 16-byte-per-lane pass over the u8 volume
// (HBM-bound; the only compulsory traffic of a TF-change LBVH rebuild).  Visibility is
// evaluated four bytes at a time with SWAR compares when the visible set is one or two bin
// intervals (ramp / band TFs), else by a 256-byte shared-memory table.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdarg>

#include "common.cuh"

namespace vs {

static __thread char g_err[512];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

// ---------------------------------------------------------------------------------------
// Visibility of four packed u8 bins.  eval<V>(x) returns a word whose bit 7 of every byte is
// that byte's visibility (other bits are don't-care unless clean<V>()).
//
//   V = 0            shared-memory table (clean)
//   V = 16           constant TF (all or nothing visible; clean)
//   V = 1 + ops      one visibility flip at bin c0        ops: bit0 c0 >= 128, bit2 bin 0 visible
//   V = 8 + ops      two flips at c0 < c1                 ops: bit1 c1 >= 128 as well
//
// Per byte, x >= c (c in [1,255]) is the high bit of (x|0x80) - (c&0x7f) OR'ed (c < 128) or
// AND'ed (c >= 128) with x; the subtraction never borrows across bytes.  So a ramp TF costs
// three integer ops per four voxels, and the OR into the running brick accumulator fuses into
// the last one (LOP3).
// ---------------------------------------------------------------------------------------
constexpr uint32_t HB = 0x80808080u;
constexpr int V_TABLE = 0, V_CONST = 16;

struct VisEval {
  uint32_t clo0, clo1, flip;
  const uint8_t* tab;  // V_TABLE: 0x80 / 0 per bin, shared memory

  template <int V>
  __device__ static constexpr bool clean() { return V == V_TABLE || V == V_CONST; }

  template <int V>
  __device__ __forceinline__ uint32_t eval(uint32_t x) const {
    if constexpr (V == V_TABLE) {
      return (uint32_t)tab[x & 0xff] | ((uint32_t)tab[(x >> 8) & 0xff] << 8) |
             ((uint32_t)tab[(x >> 16) & 0xff] << 16) | ((uint32_t)tab[x >> 24] << 24);
    } else if constexpr (V == V_CONST) {
      return flip;
    } else if constexpr (V < 8) {
      constexpr int ops = V - 1;
      const uint32_t r = (x | HB) - clo0;
      const uint32_t a = (ops & 1) ? (x & r) : (x | r);
      return (ops & 4) ? ~a : a;
    } else {
      constexpr int ops = V - 8;
      const uint32_t xh = x | HB;
      const uint32_t r0 = xh - clo0, r1 = xh - clo1;
      const uint32_t a = ((ops & 1) ? (x & r0) : (x | r0)) ^ ((ops & 2) ? (x & r1) : (x | r1));
      return (ops & 4) ? ~a : a;
    }
  }
};

__device__ __forceinline__ int load_vis(VisEval& ve, const vs_tf_params* tf, uint8_t* tab) {
  const uint32_t c0 = (uint32_t)tf->bound[0] & 0xffu, c1 = (uint32_t)tf->bound[1] & 0xffu;
  ve.clo0 = (c0 & 0x7fu) * 0x01010101u;
  ve.clo1 = (c1 & 0x7fu) * 0x01010101u;
  ve.flip = tf->start ? HB : 0u;
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    tab[b] = ((tf->vis[b >> 5] >> (b & 31)) & 1u) ? 0x80 : 0;
  ve.tab = tab;
  const int start = tf->start ? 4 : 0;
  switch (tf->mode) {
    case 1: return 1 + ((c0 & 0x80u) ? 1 : 0) + start;
    case 2: return 8 + ((c0 & 0x80u) ? 1 : 0) + ((c1 & 0x80u) ? 2 : 0) + start;
    case 3: return V_CONST;
    default: return V_TABLE;
  }
}

// 4 visible-flag bytes (0x80 each) -> 4 contiguous bits.
__device__ __forceinline__ uint32_t compress4(uint32_t g) {
  return (((g >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// ---------------------------------------------------------------------------------------
// k_brick_summary: warp task = (brick bx, brick by, 512-voxel z chunk); lane = 2 bricks in
// z (16 bytes of each z-row).  The 8x8 rows of the brick pair stream through registers; the
// 27 halo-region "any" bits are folded per row (y categories), per x slab (x categories),
// and per 4-byte word (z categories: byte 0 of the first word is z-local 0, byte 3 of the
// second word is z-local 7).
// ---------------------------------------------------------------------------------------
constexpr int SUMMARY_WARPS = 8;

// One x slab (8 rows in y) of a lane's brick pair -> 9-bit (y,z) category masks pa, pb.
template <int V, bool WRITE_BITS, bool COUNT, bool FULL>
__device__ __forceinline__ void summary_slab(const VisEval& ve, const uint8_t* __restrict__ vol,
                                             int x, int y0, int ny, int nz, int z0, int nzw,
                                             int lane, unsigned amask,
                                             uint32_t* __restrict__ bits, uint32_t& cnt,
                                             uint32_t& pa, uint32_t& pb) {
  // y-category accumulators (word pairs) for brick A and B
  uint32_t ya0 = 0, ya1 = 0, yfa0 = 0, yfa1 = 0, yla0 = 0, yla1 = 0;
  uint32_t yb0 = 0, yb1 = 0, yfb0 = 0, yfb1 = 0, ylb0 = 0, ylb1 = 0;
  const uint8_t* row = vol + ((int64_t)x * ny + y0) * nz + z0;
  uint4 v[8];
#pragma unroll
  for (int ly = 0; ly < 8; ++ly) {
    if (FULL || y0 + ly < ny)
      v[ly] = __ldcs(reinterpret_cast<const uint4*>(row + (int64_t)ly * nz));
  }
#pragma unroll
  for (int ly = 0; ly < 8; ++ly) {
    if (!(FULL || y0 + ly < ny)) continue;  // rows past ny: not part of the volume
    uint32_t g0 = ve.eval<V>(v[ly].x), g1 = ve.eval<V>(v[ly].y);
    uint32_t g2 = ve.eval<V>(v[ly].z), g3 = ve.eval<V>(v[ly].w);
    if (COUNT || WRITE_BITS) {
      if (!VisEval::clean<V>()) { g0 &= HB; g1 &= HB; g2 &= HB; g3 &= HB; }
    }
    if (COUNT) cnt += __popc(g0 | (g1 >> 1) | (g2 >> 2) | (g3 >> 3));
    if (WRITE_BITS) {
      uint32_t m = compress4(g0) | (compress4(g1) << 4) | (compress4(g2) << 8) |
                   (compress4(g3) << 12);
      uint32_t other = __shfl_down_sync(amask, m, 1);
      const int64_t wbase = ((int64_t)x * ny + (y0 + ly)) * nzw;
      if ((lane & 1) == 0) {
        uint32_t word = m | ((z0 + 16 < nz) ? (other << 16) : 0u);
        bits[wbase + (z0 >> 5)] = word;
      }
    }
    ya0 |= g0; ya1 |= g1; yb0 |= g2; yb1 |= g3;
    if (ly == 0) { yfa0 = g0; yfa1 = g1; yfb0 = g2; yfb1 = g3; }
    if (ly == 7) { yla0 = g0; yla1 = g1; ylb0 = g2; ylb1 = g3; }
  }
  if (!VisEval::clean<V>() && !(COUNT || WRITE_BITS)) {
    ya0 &= HB; ya1 &= HB; yb0 &= HB; yb1 &= HB;
    yfa0 &= HB; yfa1 &= HB; yfb0 &= HB; yfb1 &= HB;
    yla0 &= HB; yla1 &= HB; ylb0 &= HB; ylb1 &= HB;
  }
  // z categories of a word pair -> 3 bits: bit0 last slab (z7), bit1 any, bit2 first (z0)
  auto zc3 = [](uint32_t w0, uint32_t w1) -> uint32_t {
    return (w1 >> 31) | (((w0 | w1) != 0u) << 1) | (((w0 >> 7) & 1u) << 2);
  };
  pa = zc3(yla0, yla1) | (zc3(ya0, ya1) << 3) | (zc3(yfa0, yfa1) << 6);
  pb = zc3(ylb0, ylb1) | (zc3(yb0, yb1) << 3) | (zc3(yfb0, yfb1) << 6);
}

template <int V, bool WRITE_BITS, bool COUNT>
__device__ __forceinline__ void summary_body(const VisEval& ve, uint32_t* red,
                                             const uint8_t* __restrict__ vol, int nx, int ny,
                                             int nz, uint32_t* __restrict__ summary,
                                             uint32_t* __restrict__ bits,
                                             unsigned long long* __restrict__ count, int nbx,
                                             int nby, int nbz, int nzc, int64_t ntasks) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t task = (int64_t)blockIdx.x * SUMMARY_WARPS + warp;
  uint32_t cnt = 0;
  if (task < ntasks) {
    const int zc = (int)(task % nzc);
    const int64_t r = task / nzc;
    const int by = (int)(r % nby);
    const int bx = (int)(r / nby);
    const int z0 = zc * 512 + lane * 16;
    const bool active = z0 < nz;
    const int x0 = bx * 8, y0 = by * 8;
    const int nzw = (int)nzw_of(nz);
    // nz % 16 == 0, so the active lanes are a prefix of the warp (and uniform per task).
    const unsigned amask = __ballot_sync(0xffffffffu, active);

    // X-category accumulators of 9-bit (y,z) masks, per brick (A = z0..7, B = z8..15).
    uint32_t xa_any = 0, xa_first = 0, xa_last = 0;
    uint32_t xb_any = 0, xb_first = 0, xb_last = 0;
    if (active) {
      const bool full_y = y0 + 8 <= ny;  // warp-uniform
#pragma unroll 1
      for (int lx = 0; lx < 8; ++lx) {
        const int x = x0 + lx;
        if (x >= nx) break;
        uint32_t pa, pb;
        if (full_y)
          summary_slab<V, WRITE_BITS, COUNT, true>(ve, vol, x, y0, ny, nz, z0, nzw, lane,
                                                   amask, bits, cnt, pa, pb);
        else
          summary_slab<V, WRITE_BITS, COUNT, false>(ve, vol, x, y0, ny, nz, z0, nzw, lane,
                                                    amask, bits, cnt, pa, pb);
        xa_any |= pa; xb_any |= pb;
        if (lx == 0) { xa_first = pa; xb_first = pb; }
        if (lx == 7) { xa_last = pa; xb_last = pb; }
      }
      const int bz = z0 >> 3;
      const int64_t sbase = ((int64_t)bx * nby + by) * nbz;
      summary[sbase + bz] = xa_last | (xa_any << 9) | (xa_first << 18);
      if (bz + 1 < nbz) summary[sbase + bz + 1] = xb_last | (xb_any << 9) | (xb_first << 18);
    }
  }
  if (COUNT) {
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) red[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < SUMMARY_WARPS; ++w) s += red[w];
      if (s) atomicAdd(count, s);
    }
  }
}

#define VS_SUMMARY_ARGS ve, red, vol, nx, ny, nz, summary, bits, count, nbx, nby, nbz, nzc, ntasks

// Fast kernel (summary only): one instantiation per visibility shape, chosen per launch from
// the device parameter block (uniform branch), so CUDA-graph replays follow TF changes.
__global__ void __launch_bounds__(SUMMARY_WARPS * 32)
    k_brick_summary(const uint8_t* __restrict__ vol, int nx, int ny, int nz,
                    const vs_tf_params* __restrict__ tf, uint32_t* __restrict__ summary,
                    int nbx, int nby, int nbz, int nzc, int64_t ntasks) {
  __shared__ uint8_t tab[256];
  __shared__ uint32_t red[SUMMARY_WARPS];
  uint32_t* bits = nullptr;
  unsigned long long* count = nullptr;
  VisEval ve;
  const int v = load_vis(ve, tf, tab);
  __syncthreads();
  switch (v) {
    case 1: summary_body<1, false, false>(VS_SUMMARY_ARGS); break;
    case 2: summary_body<2, false, false>(VS_SUMMARY_ARGS); break;
    case 5: summary_body<5, false, false>(VS_SUMMARY_ARGS); break;
    case 6: summary_body<6, false, false>(VS_SUMMARY_ARGS); break;
    case 8: summary_body<8, false, false>(VS_SUMMARY_ARGS); break;
    case 9: summary_body<9, false, false>(VS_SUMMARY_ARGS); break;
    case 10: summary_body<10, false, false>(VS_SUMMARY_ARGS); break;
    case 11: summary_body<11, false, false>(VS_SUMMARY_ARGS); break;
    case 12: summary_body<12, false, false>(VS_SUMMARY_ARGS); break;
    case 13: summary_body<13, false, false>(VS_SUMMARY_ARGS); break;
    case 14: summary_body<14, false, false>(VS_SUMMARY_ARGS); break;
    case 15: summary_body<15, false, false>(VS_SUMMARY_ARGS); break;
    case V_CONST: summary_body<V_CONST, false, false>(VS_SUMMARY_ARGS); break;
    default: summary_body<V_TABLE, false, false>(VS_SUMMARY_ARGS); break;
  }
}

// Side-output kernel (packed undilated bits and/or the visible count): table lookup.
template <bool WRITE_BITS, bool COUNT>
__global__ void __launch_bounds__(SUMMARY_WARPS * 32)
    k_brick_summary_out(const uint8_t* __restrict__ vol, int nx, int ny, int nz,
                        const vs_tf_params* __restrict__ tf, uint32_t* __restrict__ summary,
                        uint32_t* __restrict__ bits, unsigned long long* __restrict__ count,
                        int nbx, int nby, int nbz, int nzc, int64_t ntasks) {
  __shared__ uint8_t tab[256];
  __shared__ uint32_t red[SUMMARY_WARPS];
  VisEval ve;
  load_vis(ve, tf, tab);
  __syncthreads();
  summary_body<V_TABLE, WRITE_BITS, COUNT>(VS_SUMMARY_ARGS);
}

// ---------------------------------------------------------------------------------------
// Generic classification to packed bits: thread per 32-voxel word.
// ---------------------------------------------------------------------------------------
__global__ void k_classify_bits(const uint8_t* __restrict__ vol, int nx, int ny, int nz,
                                const vs_tf_params* __restrict__ tf, uint32_t* __restrict__ bits,
                                unsigned long long* __restrict__ count) {
  __shared__ uint8_t tab[256];
  __shared__ uint32_t red[32];
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    tab[b] = (tf->vis[b >> 5] >> (b & 31)) & 1u;
  __syncthreads();
  const int64_t nzw = nzw_of(nz);
  const int64_t nwords = (int64_t)nx * ny * nzw;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t c = 0;
  if (i < nwords) {
    const int64_t rowi = i / nzw;
    const int w = (int)(i % nzw);
    const uint8_t* row = vol + rowi * nz;
    uint32_t word = 0;
    const int zend = min(32, nz - w * 32);
    for (int k = 0; k < zend; ++k) word |= (uint32_t)tab[row[w * 32 + k]] << k;
    bits[i] = word;
    c = __popc(word);
  }
  if (count) {
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
      if (s) atomicAdd(count, s);
    }
  }
}

// ---------------------------------------------------------------------------------------
// k_classify_pack<V, DIL>: classification to packed bits for rows of whole 32-voxel words
// (nz % 32 == 0, nz <= 1024), optionally fused with _dilate26 (volume.py:289-304) so the
// dilated bit volume costs one pass over the u8 volume.  Block = CP_TY output rows (+2 halo
// rows when dilating) x one CP_XC run of x slabs; warp = one row, lane = one 32-voxel word
// (two 16-byte loads, SWAR visibility).  Per x step: classify the next slab's rows, z-dilate
// with lane shuffles, y-dilate through shared memory, x-dilate with a 3-slab register ring.
// The next slab's loads are issued before the current slab is processed.
// ---------------------------------------------------------------------------------------
constexpr int CP_TY = 14, CP_XC = 64;

template <int V>
__device__ __forceinline__ uint32_t classify_word(const VisEval& ve, const uint4& a,
                                                  const uint4& b) {
  uint32_t g[8] = {ve.eval<V>(a.x), ve.eval<V>(a.y), ve.eval<V>(a.z), ve.eval<V>(a.w),
                   ve.eval<V>(b.x), ve.eval<V>(b.y), ve.eval<V>(b.z), ve.eval<V>(b.w)};
  uint32_t w = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) w |= compress4(g[k] & HB) << (4 * k);
  return w;
}

// Bulk-async (TMA, 1-D) staging of the dilating pass: a block's 16 rows of one x slab are
// CP_TY + 2 consecutive y rows = one contiguous (rows x nz)-byte run, fetched by one
// cp.async.bulk into a CP_NS-deep ring of shared-memory stages completed on mbarriers, so
// CP_NS slabs are in flight per block without holding them in registers.
#ifndef VS_CP_BULK
#define VS_CP_BULK 1
#endif
#ifndef VS_CP_NS
#define VS_CP_NS 4
#endif
constexpr int CP_NS = VS_CP_NS;
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int V, bool DIL>
__device__ __forceinline__ void classify_pack_body(const VisEval& ve, uint32_t* zs,
                                                   uint32_t* red, const uint8_t* __restrict__ vol,
                                                   int nx, int ny, int nz,
                                                   uint32_t* __restrict__ out,
                                                   unsigned long long* __restrict__ count,
                                                   int* __restrict__ bbox) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nzw = nz >> 5;
  const int ty = DIL ? CP_TY : (int)(blockDim.x >> 5);
  const int y0 = blockIdx.x * ty, x0 = blockIdx.y * CP_XC;
  const int xe = min(nx, x0 + CP_XC);
  const int y = y0 + warp - (DIL ? 1 : 0);
  const bool rowok = y >= 0 && y < ny && lane < nzw;
  const bool outrow = rowok && (!DIL || (warp >= 1 && warp <= CP_TY));
  const uint8_t* rowp = vol + (int64_t)y * nz + lane * 32;
  const int64_t xstride = (int64_t)ny * nz;
  auto load = [&](int x, uint4& a, uint4& b) {
    if (rowok && x >= 0 && x < nx) {
      const uint4* q = reinterpret_cast<const uint4*>(rowp + (int64_t)x * xstride);
      a = __ldcs(q);
      b = __ldcs(q + 1);
    }
  };
  uint32_t cnt = 0;
  uint4 a = make_uint4(0, 0, 0, 0), b = a, na = a, nb = a;
  if (!DIL) {
    load(x0, a, b);
    for (int x = x0; x < xe; ++x) {
      if (x + 1 < xe) load(x + 1, na, nb);
      if (outrow) {
        const uint32_t w = classify_word<V>(ve, a, b);
        out[((int64_t)x * ny + y) * nzw + lane] = w;
        cnt += __popc(w);
      }
      a = na;
      b = nb;
    }
  } else {
    // y/z-dilated words of slabs x-1, x (ring), output row = warp
    uint32_t prev = 0, cur = 0;
    // tight box of the dilated flags (shrink_to_occupied of the whole volume, the k-d root,
    // kdtree.py:398) as a by-product: x / z extremes of this thread's output words
    int bx0 = 0x3fffffff, bx1 = -1, bz0 = 0x3fffffff, bz1 = -1;
#if VS_CP_BULK
    // slab xs = x0 - 1 + j lives in stage j % CP_NS; the block's rows [ylo, yhi) are one
    // contiguous run per slab.  Slabs outside [0, nx) complete their phase by a plain arrive.
    extern __shared__ __align__(128) uint8_t cp_stage[];
    uint64_t* full = reinterpret_cast<uint64_t*>(cp_stage);
    uint8_t* stage0 = cp_stage + 128;
    const int ylo = max(y0 - 1, 0), yhi = min(y0 + CP_TY + 1, ny);
    const uint32_t run = (uint32_t)(yhi - ylo) * (uint32_t)nz;
    const size_t stage_bytes = (size_t)(CP_TY + 2) * nz;
    const int nj = xe - x0 + 2;  // slabs x0 - 1 .. xe
    auto issue = [&](int j) {
      const int xsj = x0 - 1 + j;
      uint64_t* bar = full + (j % CP_NS);
      if (xsj >= 0 && xsj < nx)
        bulk_load(stage0 + (size_t)(j % CP_NS) * stage_bytes,
                  vol + ((int64_t)xsj * ny + ylo) * nz, run, bar);
      else
        mbar_arrive(bar);
    };
    if (threadIdx.x == 0) {
      for (int k = 0; k < CP_NS; ++k) mbar_init(full + k, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 0; j < min(CP_NS, nj); ++j) issue(j);
    const uint8_t* srow = stage0 + (size_t)(y - ylo) * nz + lane * 32;
    for (int xs = x0 - 1; xs <= xe; ++xs) {
      const int j = xs - (x0 - 1);
      mbar_wait(full + (j % CP_NS), (uint32_t)(j / CP_NS) & 1u);
      uint32_t w = 0;
      if (rowok && xs >= 0 && xs < nx) {
        const uint4* q = reinterpret_cast<const uint4*>(srow + (size_t)(j % CP_NS) * stage_bytes);
        w = classify_word<V>(ve, q[0], q[1]);
      }
#else
    // three slabs in flight ahead of the one being classified; the y-dilation exchange is
    // double-buffered so one barrier per slab suffices
    uint4 fa = make_uint4(0, 0, 0, 0), fb = fa, ga = fa, gb = fa;
    load(x0 - 1, a, b);
    load(x0, na, nb);
    load(x0 + 1, fa, fb);
    for (int xs = x0 - 1; xs <= xe; ++xs) {
      // slab xs: classify, count, z-dilate, y-dilate
      ga = make_uint4(0, 0, 0, 0);
      gb = ga;
      if (xs + 3 <= xe) load(xs + 3, ga, gb);
      uint32_t w = 0;
      if (rowok && xs >= 0 && xs < nx) w = classify_word<V>(ve, a, b);
#endif
      if (outrow && xs >= x0 && xs < xe) cnt += __popc(w);
      const uint32_t up = __shfl_up_sync(0xffffffffu, w, 1);
      const uint32_t dn = __shfl_down_sync(0xffffffffu, w, 1);
      uint32_t zd = w | (w << 1) | (w >> 1);
      if (lane > 0) zd |= up >> 31;
      if (lane + 1 < nzw) zd |= dn << 31;
      uint32_t* zb = zs + (xs & 1) * ((CP_TY + 2) * 32);
      zb[warp * 32 + lane] = zd;
      __syncthreads();
#if VS_CP_BULK
      // every thread is done with stage j: refill it with slab j + CP_NS
      if (threadIdx.x == 0 && j + CP_NS < nj) issue(j + CP_NS);
#endif
      uint32_t yd = 0;
      if (warp >= 1 && warp <= CP_TY) yd = zb[(warp - 1) * 32 + lane] | zd | zb[(warp + 1) * 32 + lane];
      // slab xs - 1 is complete: prev (xs-2) | cur (xs-1) | yd (xs)
      if (outrow && xs - 1 >= x0) {
        const uint32_t dw = prev | cur | yd;
        out[((int64_t)(xs - 1) * ny + y) * nzw + lane] = dw;
        if (dw) {
          bx0 = min(bx0, xs - 1);
          bx1 = xs - 1;
          bz0 = min(bz0, 32 * lane + __ffs(dw) - 1);
          bz1 = max(bz1, 32 * lane + 31 - __clz(dw));
        }
      }
      prev = cur;
      cur = yd;
#if !VS_CP_BULK
      a = na; b = nb;
      na = fa; nb = fb;
      fa = ga; fb = gb;
#endif
    }
    if (bbox) {
      bx0 = __reduce_min_sync(0xffffffffu, bx0);
      bx1 = __reduce_max_sync(0xffffffffu, bx1);
      bz0 = __reduce_min_sync(0xffffffffu, bz0);
      bz1 = __reduce_max_sync(0xffffffffu, bz1);
      if (lane == 0 && bx1 >= 0) {  // few warps see flags: global atomics per warp
        atomicMin(bbox + 0, bx0); atomicMax(bbox + 3, bx1 + 1);
        atomicMin(bbox + 1, y);   atomicMax(bbox + 4, y + 1);
        atomicMin(bbox + 2, bz0); atomicMax(bbox + 5, bz1 + 1);
      }
    }
  }
  if (count) {
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) red[warp] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
      if (s) atomicAdd(count, s);
    }
  }
}

#define VS_CP_ARGS ve, zs, red, vol, nx, ny, nz, out, count, bbox

template <bool DIL>
__global__ void __launch_bounds__(1024) k_classify_pack(const uint8_t* __restrict__ vol, int nx,
                                                        int ny, int nz,
                                                        const vs_tf_params* __restrict__ tf,
                                                        uint32_t* __restrict__ out,
                                                        unsigned long long* __restrict__ count,
                                                        int* __restrict__ bbox) {
  __shared__ uint8_t tab[256];
  __shared__ uint32_t zs[2 * (CP_TY + 2) * 32];
  __shared__ uint32_t red[32];
  VisEval ve;
  const int v = load_vis(ve, tf, tab);
  __syncthreads();
  switch (v) {
    case 1: classify_pack_body<1, DIL>(VS_CP_ARGS); break;
    case 2: classify_pack_body<2, DIL>(VS_CP_ARGS); break;
    case 5: classify_pack_body<5, DIL>(VS_CP_ARGS); break;
    case 6: classify_pack_body<6, DIL>(VS_CP_ARGS); break;
    case 8: classify_pack_body<8, DIL>(VS_CP_ARGS); break;
    case 9: classify_pack_body<9, DIL>(VS_CP_ARGS); break;
    case 10: classify_pack_body<10, DIL>(VS_CP_ARGS); break;
    case 11: classify_pack_body<11, DIL>(VS_CP_ARGS); break;
    case 12: classify_pack_body<12, DIL>(VS_CP_ARGS); break;
    case 13: classify_pack_body<13, DIL>(VS_CP_ARGS); break;
    case 14: classify_pack_body<14, DIL>(VS_CP_ARGS); break;
    case 15: classify_pack_body<15, DIL>(VS_CP_ARGS); break;
    case V_CONST: classify_pack_body<V_CONST, DIL>(VS_CP_ARGS); break;
    default: classify_pack_body<V_TABLE, DIL>(VS_CP_ARGS); break;
  }
}

// Empty tight box {FAR, FAR, FAR, -1, -1, -1} for the atomic min / max of k_classify_pack.
__global__ void k_bbox_init(int* __restrict__ bbox) {
  if (threadIdx.x < 6) bbox[threadIdx.x] = threadIdx.x < 3 ? 0x3fffffff : -1;
}

__global__ void k_quantize(const float* __restrict__ f, int64_t n, uint8_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // volume.py:159-162 in float64, no FMA: floor(v*255 + 0.5), clip [0, 255]; NaN -> 0 like
  // numpy's int64 cast of NaN (INT64_MIN) clipped to 0.
  double d = floor(__dadd_rn(__dmul_rn((double)f[i], 255.0), 0.5));
  int q = (d != d) ? 0 : (d < 0.0 ? 0 : (d > 255.0 ? 255 : (int)d));
  out[i] = (uint8_t)q;
}

// Row-dilated word: z dilation within a packed row, border-clipped.
__device__ __forceinline__ uint32_t zdil(const uint32_t* __restrict__ row, int w, int nzw,
                                         uint32_t lastmask) {
  uint32_t v = __ldg(row + w);
  uint32_t r = v | (v << 1) | (v >> 1);
  if (w > 0) r |= __ldg(row + w - 1) >> 31;
  if (w + 1 < nzw) r |= __ldg(row + w + 1) << 31;
  if (w + 1 == nzw) r &= lastmask;
  return r;
}

// _dilate26 on packed bits: thread = (word w, row y, x chunk); slides along x keeping the
// y/z-dilated rows x-1, x, x+1 in registers.
constexpr int DIL_XCHUNK = 16;
__global__ void k_dilate(const uint32_t* __restrict__ in, int nx, int ny, int nz,
                         uint32_t* __restrict__ out) {
  const int nzw = (int)nzw_of(nz);
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int x0 = blockIdx.z * DIL_XCHUNK;
  if (w >= nzw) return;
  const uint32_t lastmask = (nz & 31) ? ((1u << (nz & 31)) - 1u) : 0xffffffffu;
  auto yz = [&](int x) -> uint32_t {
    if (x < 0 || x >= nx) return 0u;
    uint32_t r = 0;
    for (int dy = -1; dy <= 1; ++dy) {
      int yy = y + dy;
      if (yy < 0 || yy >= ny) continue;
      r |= zdil(in + ((int64_t)x * ny + yy) * nzw, w, nzw, lastmask);
    }
    return r;
  };
  uint32_t prev = yz(x0 - 1), cur = yz(x0);
  const int xe = min(nx, x0 + DIL_XCHUNK);
  for (int x = x0; x < xe; ++x) {
    uint32_t nxt = yz(x + 1);
    out[((int64_t)x * ny + y) * nzw + w] = prev | cur | nxt;
    prev = cur;
    cur = nxt;
  }
}

__global__ void k_pack(const uint8_t* __restrict__ b, int64_t nrows, int nz,
                       uint32_t* __restrict__ bits) {
  const int64_t nzw = nzw_of(nz);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows * nzw) return;
  const int64_t r = i / nzw;
  const int w = (int)(i % nzw);
  const uint8_t* row = b + r * nz + w * 32;
  const int zend = min(32, nz - w * 32);
  uint32_t word = 0;
  for (int k = 0; k < zend; ++k) word |= (row[k] ? 1u : 0u) << k;
  bits[i] = word;
}

__global__ void k_unpack(const uint32_t* __restrict__ bits, int64_t nrows, int nz,
                         uint8_t* __restrict__ b) {
  const int64_t n = nrows * nz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = i / nz;
  const int z = (int)(i % nz);
  b[i] = (bits[r * nzw_of(nz) + (z >> 5)] >> (z & 31)) & 1u;
}

__global__ void k_count_bits(const uint32_t* __restrict__ bits, int64_t nwords,
                             unsigned long long* __restrict__ count) {
  __shared__ uint32_t red[32];
  uint32_t c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords;
       i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(bits[i]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    if (s) atomicAdd(count, s);
  }
}

// Per-cell vote, thread per cell (C-order), early exit on the first set word.
__global__ void k_vote_cells(const uint32_t* __restrict__ bits, int nx, int ny, int nz, int cs,
                             int ncx, int ncy, int ncz, uint8_t* __restrict__ flags) {
  const int64_t ncell = (int64_t)ncx * ncy * ncz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncell) return;
  const int cz = (int)(i % ncz);
  const int cy = (int)((i / ncz) % ncy);
  const int cx = (int)(i / ((int64_t)ncz * ncy));
  const int nzw = (int)nzw_of(nz);
  const int xa = cx * cs, xb = min(nx, xa + cs);
  const int ya = cy * cs, yb = min(ny, ya + cs);
  const int za = cz * cs, zb = min(nz, za + cs);
  const int wa = za >> 5, wb = (zb - 1) >> 5;
  uint8_t f = 0;
  for (int x = xa; x < xb && !f; ++x)
    for (int y = ya; y < yb && !f; ++y) {
      const uint32_t* row = bits + ((int64_t)x * ny + y) * nzw;
      for (int w = wa; w <= wb; ++w) {
        uint32_t m = 0xffffffffu;
        if (w == wa) m &= 0xffffffffu << (za & 31);
        if (w == wb && ((zb & 31) != 0)) m &= (1u << (zb & 31)) - 1u;
        if (__ldg(row + w) & m) { f = 1; break; }
      }
    }
  flags[i] = f;
}

// 16^3 cell votes when every row is whole words (nz % 32 == 0, nz <= 1024 -> <= 64 cells in
// z): block per (cx, cy) cell column, thread per row of the column's 16 x 16 footprint, the
// row read with 16-byte loads (all in flight), a 64-bit z-cell mask per thread OR-reduced.
__global__ void __launch_bounds__(256) k_vote_cells16(const uint32_t* __restrict__ bits, int nx,
                                                      int ny, int nz, int ncy, int ncz,
                                                      uint8_t* __restrict__ flags) {
  __shared__ unsigned long long red[8];
  const int cx = blockIdx.x / ncy, cy = blockIdx.x - (blockIdx.x / ncy) * ncy;
  const int x = cx * 16 + (threadIdx.x >> 4), y = cy * 16 + (threadIdx.x & 15);
  const int nzw = nz >> 5;
  unsigned long long m = 0;
  if (x < nx && y < ny) {
    const uint4* row = reinterpret_cast<const uint4*>(bits + ((int64_t)x * ny + y) * nzw);
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 4 * k < nzw ? __ldg(row + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int wi = 4 * k + j;  // word index: cells 2 wi (bits 0-15), 2 wi + 1 (bits 16-31)
        m |= (unsigned long long)((w[j] & 0xffffu) != 0u) << (2 * wi);
        m |= (unsigned long long)((w[j] >> 16) != 0u) << (2 * wi + 1);
      }
    }
  }
  for (int o = 16; o; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < ncz) {
    unsigned long long t = 0;
    for (int k = 0; k < 8; ++k) t |= red[k];
    flags[((int64_t)cx * ncy + cy) * ncz + threadIdx.x] = (t >> threadIdx.x) & 1ull;
  }
}

// ---------------------------------------------------------------------------------------
// Summary -> Morton bitmap (+ tile counts, + 16^3 cells).  CTA = one 8^3 tile of bricks =
// one aligned 512-code Morton range; the 10^3 summary halo is staged in shared memory.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int sbit(int ex, int ey, int ez) {
  return (ex + 1) * 9 + (ey + 1) * 3 + (ez + 1);
}

__global__ void __launch_bounds__(512)
    k_summary_to_bitmap(const uint32_t* __restrict__ summary, int nbx, int nby, int nbz,
                        int dilate, uint32_t* __restrict__ bitmap,
                        uint32_t* __restrict__ tile_counts, uint8_t* __restrict__ cell16,
                        int ncx, int ncy, int ncz) {
  __shared__ uint32_t s[10][10][10];
  __shared__ uint32_t wc[16];
  const uint32_t tile = blockIdx.x;
  const int tx = (int)compact10(tile) * 8, ty = (int)compact10(tile >> 1) * 8,
            tz = (int)compact10(tile >> 2) * 8;
  const int t = threadIdx.x;
  if (tx >= nbx || ty >= nby || tz >= nbz) {  // tile outside the brick grid
    if (t < 16) bitmap[(size_t)tile * 16 + t] = 0;
    if (t == 0) tile_counts[tile] = 0;
    return;
  }
  for (int k = t; k < 1000; k += 512) {
    const int hx = k / 100, hy = (k / 10) % 10, hz = k % 10;
    const int gx = tx + hx - 1, gy = ty + hy - 1, gz = tz + hz - 1;
    uint32_t v = 0;
    if (gx >= 0 && gx < nbx && gy >= 0 && gy < nby && gz >= 0 && gz < nbz)
      v = summary[((int64_t)gx * nby + gy) * nbz + gz];
    s[hx][hy][hz] = v;
  }
  __syncthreads();
  const int lx = (int)compact10((uint32_t)t), ly = (int)compact10((uint32_t)t >> 1),
            lz = (int)compact10((uint32_t)t >> 2);
  const int bx = tx + lx, by = ty + ly, bz = tz + lz;
  uint32_t f = 0;
  if (bx < nbx && by < nby && bz < nbz) {
    if (dilate) {
#pragma unroll
      for (int ex = -1; ex <= 1; ++ex)
#pragma unroll
        for (int ey = -1; ey <= 1; ++ey)
#pragma unroll
          for (int ez = -1; ez <= 1; ++ez)
            f |= s[lx + 1 + ex][ly + 1 + ey][lz + 1 + ez] >> sbit(ex, ey, ez);
      f &= 1u;
    } else {
      f = (s[lx + 1][ly + 1][lz + 1] >> sbit(0, 0, 0)) & 1u;
    }
  }
  const uint32_t ball = __ballot_sync(0xffffffffu, f != 0);
  const int lane = t & 31, warp = t >> 5;
  if (lane == 0) {
    bitmap[(size_t)tile * 16 + warp] = ball;
    wc[warp] = __popc(ball);
  }
  if (cell16 && (lane & 7) == 0) {
    const int cx = bx >> 1, cy = by >> 1, cz = bz >> 1;
    if (cx < ncx && cy < ncy && cz < ncz)
      cell16[((int64_t)cx * ncy + cy) * ncz + cz] = ((ball >> lane) & 0xffu) ? 1 : 0;
  }
  __syncthreads();
  if (t == 0) {
    uint32_t c = 0;
    for (int k = 0; k < 16; ++k) c += wc[k];
    tile_counts[tile] = c;
  }
}

// ---------------------------------------------------------------------------------------
// Brick flags of one 512-code Morton tile (8^3 bricks) -> Morton bitmap words, tile count,
// optional 16^3 cells and optional C-order leaf-brick bit grid.  Persistent CTAs; the next
// tile's inputs are loaded into registers before the current tile is processed.
//   FL_SUMMARY / FL_SUMMARY_DILATE: from the 27-bit summaries.  The dilated vote
//     flag(b) = OR_e bit sbit(e) of S[b + e] is evaluated separably in shared memory:
//     U = OR over ex (9 bits per brick), V = OR over ey (3 bits), flag = OR over ez.
//   FL_PRESENCE: from the per-volume 256-bit halo presence masks (vs_presence_build):
//     flag(b) = OR over channels of (presence_c[b] & vis_c) != 0 -- exact, because a brick's
//     dilated vote is the OR of base visibility over its 1-voxel halo (volume.py:289-319,
//     lbvh.py:93-96), and visibility depends on the bin alone.
// ---------------------------------------------------------------------------------------
enum { FL_SUMMARY = 0, FL_SUMMARY_DILATE = 1, FL_PRESENCE = 2 };
constexpr int FL_T = 256;

template <int MODE>
__global__ void __launch_bounds__(FL_T)
    k_flags_tiles(const uint32_t* __restrict__ src, const uint32_t* const* __restrict__ chans,
                  const int32_t* __restrict__ tf_params,
                  int nch, int nbx, int nby, int nbz, int64_t ntiles,
                  uint32_t* __restrict__ bitmap, uint32_t* __restrict__ tile_counts,
                  uint8_t* __restrict__ cell16, int ncx, int ncy, int ncz,
                  uint32_t* __restrict__ grid) {
  __shared__ uint32_t S[1000];
  __shared__ uint32_t U[800];
  __shared__ uint8_t V[640];
  __shared__ uint8_t F[512];
  __shared__ uint32_t s_vis[4][8];
  __shared__ uint32_t s_wc[16];  // popcount of each of the tile's 16 bitmap words
  const int t = threadIdx.x, lane = t & 31;
  if (MODE == FL_PRESENCE && t < 32 && t < 8 * nch) s_vis[t >> 3][t & 7] = tf_params[16 * (t >> 3) + (t & 7)];
  constexpr int NL = MODE == FL_SUMMARY_DILATE ? 4 : 2;  // halo words / bricks per thread
  // the thread's two bricks of a tile (Morton ranks t and t + FL_T): tile-invariant offsets
  int loc[2][3];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t m = (uint32_t)(t + q * FL_T);
    loc[q][0] = (int)compact10(m);
    loc[q][1] = (int)compact10(m >> 1);
    loc[q][2] = (int)compact10(m >> 2);
  }
  uint32_t reg[NL][MODE == FL_PRESENCE ? 8 : 1];
  auto tile_origin = [](int64_t tile, int& tx, int& ty, int& tz) {
    tx = (int)compact10((uint32_t)tile) * 8;
    ty = (int)compact10((uint32_t)tile >> 1) * 8;
    tz = (int)compact10((uint32_t)tile >> 2) * 8;
  };
  auto load = [&](int64_t tile) {
    int tx, ty, tz;
    tile_origin(tile, tx, ty, tz);
    if (tx >= nbx || ty >= nby || tz >= nbz) return;
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      if (MODE == FL_SUMMARY_DILATE) {
        const int k = t + q * FL_T;
        uint32_t v = 0;
        if (k < 1000) {
          const int gx = tx + k / 100 - 1, gy = ty + (k / 10) % 10 - 1, gz = tz + k % 10 - 1;
          if (gx >= 0 && gx < nbx && gy >= 0 && gy < nby && gz >= 0 && gz < nbz)
            v = __ldg(src + ((int64_t)gx * nby + gy) * nbz + gz);
        }
        reg[q][0] = v;
      } else {
        const int bx = tx + loc[q][0], by = ty + loc[q][1], bz = tz + loc[q][2];
        const bool in = bx < nbx && by < nby && bz < nbz;
        const int64_t lin = ((int64_t)bx * nby + by) * nbz + bz;
        if (MODE == FL_SUMMARY) {
          reg[q][0] = in ? __ldg(src + lin) : 0u;
        } else {
          uint32_t f = 0;  // channels > 1: folded to the flag here (masks in shared memory)
          for (int c = 0; c < nch; ++c) {
            uint4 a = make_uint4(0, 0, 0, 0), b = a;
            if (in) {
              const uint4* pp = reinterpret_cast<const uint4*>(chans[c] + lin * 8);
              a = __ldg(pp);
              b = __ldg(pp + 1);
            }
            if (nch == 1) {
              reg[q][0] = a.x; reg[q][1] = a.y; reg[q][2] = a.z; reg[q][3] = a.w;
              reg[q][4] = b.x; reg[q][5] = b.y; reg[q][6] = b.z; reg[q][7] = b.w;
            } else {
              f |= (a.x & s_vis[c][0]) | (a.y & s_vis[c][1]) | (a.z & s_vis[c][2]) |
                   (a.w & s_vis[c][3]) | (b.x & s_vis[c][4]) | (b.y & s_vis[c][5]) |
                   (b.z & s_vis[c][6]) | (b.w & s_vis[c][7]);
            }
          }
          if (nch > 1) reg[q][0] = f ? 1u : 0u;
        }
      }
    }
  };
  __syncthreads();
  int64_t tile = blockIdx.x;
  if (tile < ntiles) load(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    __syncthreads();  // the previous tile's shared-memory readers are done
    int tx, ty, tz;
    tile_origin(tile, tx, ty, tz);
    const bool inside = tx < nbx && ty < nby && tz < nbz;  // CTA-uniform
    uint32_t flag[2] = {0u, 0u};
    if (inside) {
      if (MODE == FL_SUMMARY_DILATE) {
#pragma unroll
        for (int q = 0; q < NL; ++q)
          if (t + q * FL_T < 1000) S[t + q * FL_T] = reg[q][0];
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (MODE == FL_SUMMARY) {
            flag[q] = (reg[q][0] >> 13) & 1u;  // sbit(0,0,0): the brick itself
          } else if (nch > 1) {
            flag[q] = reg[q][0];
          } else {
            uint32_t any = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) any |= reg[q][w] & s_vis[0][w];
            flag[q] = any != 0u;
          }
        }
      }
    }
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) load(next);  // in flight while this tile is processed
    if (!inside) {
      if (t < 16) bitmap[tile * 16 + t] = 0;
      if (t == 0) tile_counts[tile] = 0;
      continue;
    }
    if (MODE == FL_SUMMARY_DILATE) {
      __syncthreads();  // S stored
      for (int k = t; k < 800; k += FL_T) {  // U[x][y][z], x in 0..7, y, z in halo 0..9
        const int x = k / 100, yz = k - x * 100;
        U[k] = (S[x * 100 + yz] | (S[(x + 1) * 100 + yz] >> 9) | (S[(x + 2) * 100 + yz] >> 18)) &
               0x1FFu;
      }
      __syncthreads();
      for (int k = t; k < 640; k += FL_T) {  // V[x][y][z], y in 0..7, z in halo 0..9
        const int x = k / 80, r = k - x * 80, y = r / 10, z = r - y * 10;
        const int u = x * 100 + y * 10 + z;
        V[k] = (uint8_t)((U[u] | (U[u + 10] >> 3) | (U[u + 20] >> 6)) & 7u);
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int v = loc[q][0] * 80 + loc[q][1] * 10 + loc[q][2];
        flag[q] = ((V[v] & 1u) | ((V[v + 1] >> 1) & 1u) | ((V[v + 2] >> 2) & 1u));
      }
    }
    // bricks outside the grid (partial tiles) never vote
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t m = (uint32_t)(t + q * FL_T);
      const int lx = loc[q][0], ly = loc[q][1], lz = loc[q][2];
      const bool in = tx + lx < nbx && ty + ly < nby && tz + lz < nbz;
      flag[q] = in ? flag[q] : 0u;
      const uint32_t ball = __ballot_sync(0xffffffffu, flag[q] != 0u);
      const int wd = (int)(m >> 5);
      if (lane == 0) {
        bitmap[tile * 16 + wd] = ball;
        s_wc[wd] = (uint32_t)__popc(ball);
      }
      if (cell16 && (lane & 7) == 0) {
        const int cx = (tx + lx) >> 1, cy = (ty + ly) >> 1, cz = (tz + lz) >> 1;
        if (cx < ncx && cy < ncy && cz < ncz)
          cell16[((int64_t)cx * ncy + cy) * ncz + cz] = ((ball >> lane) & 0xffu) ? 1 : 0;
      }
      if (grid) F[(lx * 8 + ly) * 8 + lz] = (uint8_t)(flag[q] != 0u);
    }
    __syncthreads();
    if (t == 0) {
      uint32_t c = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) c += s_wc[k];
      tile_counts[tile] = c;
    }
    if (grid && t < 64) {  // C-order leaf-brick bits: one byte per (x, y) row of 8 z-bricks
      const int lx = t >> 3, ly = t & 7, bx = tx + lx, by = ty + ly;
      if (bx < nbx && by < nby) {
        uint32_t byte = 0;
#pragma unroll
        for (int z = 0; z < 8; ++z) byte |= (uint32_t)F[t * 8 + z] << z;
        const int64_t lin = ((int64_t)bx * nby + by) * nbz + tz;
        if ((nbz & 7) == 0) {
          reinterpret_cast<uint8_t*>(grid)[lin >> 3] = (uint8_t)byte;
        } else {
          for (int z = 0; z < 8; ++z)
            if ((byte >> z) & 1u) atomicOr(grid + ((lin + z) >> 5), 1u << ((lin + z) & 31));
        }
      }
    }
  }
}

// The warm vote straight from the presence masks in C order (no cells requested, nbz % 32 == 0):
// CTA per brick row (bx, by), thread per bz.  Loads are one 32-byte mask per thread, row-
// contiguous; the renderer's C-order brick bits are the warps' ballots; the Morton bitmap and its
// tile counts (pre-zeroed) take one atomicOr / atomicAdd per flagged brick (~10% of them).
__global__ void __launch_bounds__(256)
    k_presence_vote(const uint32_t* const* __restrict__ chans,
                    const int32_t* __restrict__ tf_params, int nch, int nby, int nbz,
                    uint32_t* __restrict__ bitmap, uint32_t* __restrict__ tile_counts,
                    uint32_t* __restrict__ grid) {
  __shared__ uint32_t s_vis[4][8];
  const int t = threadIdx.x;
  if (t < 8 * nch) s_vis[t >> 3][t & 7] = tf_params[16 * (t >> 3) + (t & 7)];
  __syncthreads();
  const int row = blockIdx.y, bx = row / nby, by = row - (row / nby) * nby;
  const int bz = blockIdx.x * blockDim.x + t;
  uint32_t f = 0;
  const int64_t lin = (int64_t)row * nbz + bz;
  if (bz < nbz) {
    for (int c = 0; c < nch; ++c) {
      const uint4* pp = reinterpret_cast<const uint4*>(chans[c] + lin * 8);
      const uint4 a = __ldcs(pp), b = __ldcs(pp + 1);
      f |= (a.x & s_vis[c][0]) | (a.y & s_vis[c][1]) | (a.z & s_vis[c][2]) |
           (a.w & s_vis[c][3]) | (b.x & s_vis[c][4]) | (b.y & s_vis[c][5]) |
           (b.z & s_vis[c][6]) | (b.w & s_vis[c][7]);
    }
  }
  const uint32_t ball = __ballot_sync(0xffffffffu, f != 0u);
  if (grid && (t & 31) == 0 && bz < nbz) grid[lin >> 5] = ball;
  if (f) {
    const uint32_t code = spread10((uint32_t)bx) | (spread10((uint32_t)by) << 1) |
                          (spread10((uint32_t)bz) << 2);
    atomicOr(bitmap + (code >> 5), 1u << (code & 31));
    atomicAdd(tile_counts + (code >> 9), 1u);
  }
}

// Per-volume 256-bit presence mask of every 8^3 brick's 1-voxel halo (the TF-independent warm
// path of the brick vote: a TF change then reads 32 B per brick instead of the volume).  CTA
// per (bx, by) brick column; each thread takes 16-byte z chunks of the column's 10 x 10 halo
// rows; a byte sets its bit in the mask of its brick and, at a brick face, of the z neighbour
// whose halo it is.  Bits are tested before the shared atomic, so repeated values are cheap.
constexpr int PR_T = 256;
__global__ void __launch_bounds__(PR_T)
    k_presence(const uint8_t* __restrict__ vol, int nx, int ny, int nz, int nby, int nbz,
               int bx0, uint32_t* __restrict__ presence) {
  extern __shared__ uint32_t pm[];  // nbz * 8 words
  const int bx = bx0 + (int)(blockIdx.x / nby), by = blockIdx.x - (blockIdx.x / nby) * nby;
  for (int k = threadIdx.x; k < nbz * 8; k += PR_T) pm[k] = 0;
  __syncthreads();
  const int x0 = max(bx * 8 - 1, 0), x1 = min(bx * 8 + 9, nx);
  const int y0 = max(by * 8 - 1, 0), y1 = min(by * 8 + 9, ny);
  const int nyr = y1 - y0, nchunk = nz >> 4;
  const int total = (x1 - x0) * nyr * nchunk;
  auto set = [&](int brick, uint32_t v) {
    uint32_t* w = pm + brick * 8 + (v >> 5);
    const uint32_t bit = 1u << (v & 31);
    if (!(*w & bit)) atomicOr(w, bit);
  };
  // k = r * nchunk + c walks the column's rows x chunks; (x, y, c) advance incrementally
  const int step_r = PR_T / nchunk, step_c = PR_T % nchunk;
  int c = threadIdx.x % nchunk, r = threadIdx.x / nchunk;
  int x = x0 + r / nyr, y = y0 + r % nyr;
  for (int k = threadIdx.x; k < total; k += PR_T) {
    const uint4 q = __ldcs(reinterpret_cast<const uint4*>(vol + ((int64_t)x * ny + y) * nz) + c);
    const int b0 = 2 * c;  // bricks b0 (bytes 0-7) and b0 + 1 (bytes 8-15)
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    if ((q.x | q.y) == 0u) {
      set(b0, 0u);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) set(b0, (w[j >> 2] >> (8 * (j & 3))) & 0xffu);
    }
    if ((q.z | q.w) == 0u) {
      set(b0 + 1, 0u);
    } else {
#pragma unroll
      for (int j = 8; j < 16; ++j) set(b0 + 1, (w[j >> 2] >> (8 * (j & 3))) & 0xffu);
    }
    // z halo: byte 0 belongs to brick b0 - 1's halo, byte 7 to b0 + 1's, byte 8 to b0's,
    // byte 15 to b0 + 2's
    if (b0 > 0) set(b0 - 1, q.x & 0xffu);
    set(b0 + 1, q.y >> 24);
    set(b0, q.z & 0xffu);
    if (b0 + 2 < nbz) set(b0 + 2, q.w >> 24);
    c += step_c;
    int dr = step_r;
    if (c >= nchunk) { c -= nchunk; ++dr; }
    y += dr;
    while (y >= y1) { y -= nyr; ++x; }
  }
  __syncthreads();
  uint32_t* out = presence + (((int64_t)bx * nby + by) * nbz) * 8;
  for (int k = threadIdx.x; k < nbz * 8; k += PR_T) out[k] = pm[k];
}

__global__ void k_flags_scatter(const uint8_t* __restrict__ flags, int nbx, int nby, int nbz,
                                uint32_t* __restrict__ bitmap) {
  const int64_t n = (int64_t)nbx * nby * nbz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  const uint32_t bz = (uint32_t)(i % nbz), by = (uint32_t)((i / nbz) % nby),
                 bx = (uint32_t)(i / ((int64_t)nbz * nby));
  const uint32_t code = morton3(bx, by, bz);
  atomicOr(bitmap + (code >> 5), 1u << (code & 31));
}

__global__ void k_tile_counts(const uint32_t* __restrict__ bitmap, int64_t ntiles,
                              uint32_t* __restrict__ tile_counts) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  uint32_t c = 0;
  const uint4* p = reinterpret_cast<const uint4*>(bitmap + t * 16);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint4 v = p[k];
    c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  }
  tile_counts[t] = c;
}

__global__ void k_bitmap_to_scan_flags(const uint32_t* __restrict__ bitmap, int nbx, int nby,
                                       int nbz, uint8_t* __restrict__ flags) {
  const int64_t n = (int64_t)nbx * nby * nbz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t bz = (uint32_t)(i % nbz), by = (uint32_t)((i / nbz) % nby),
                 bx = (uint32_t)(i / ((int64_t)nbz * nby));
  const uint32_t code = morton3(bx, by, bz);
  flags[i] = (bitmap[code >> 5] >> (code & 31)) & 1u;
}

__global__ void k_decode_scan(const int64_t* __restrict__ idx, const int* __restrict__ n_dev,
                              int nby, int nbz, int32_t* __restrict__ coords,
                              uint32_t* __restrict__ codes, int64_t cap) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= cap || k >= *n_dev) return;
  const int64_t i = idx[k];
  const int bz = (int)(i % nbz), by = (int)((i / nbz) % nby), bx = (int)(i / ((int64_t)nbz * nby));
  coords[3 * k] = bx;
  coords[3 * k + 1] = by;
  coords[3 * k + 2] = bz;
  codes[k] = morton3(bx, by, bz);
}

}  // namespace vs

using namespace vs;

// =======================================================================================
// C ABI
// =======================================================================================
extern "C" {

const char* vs_version(void) { return "vsb200 0.1 sm_100a"; }

int vs_last_error(char* buf, size_t size) {
  if (buf && size) {
    strncpy(buf, g_err, size - 1);
    buf[size - 1] = 0;
  }
  return (int)strlen(g_err);
}

int vs_tf_params_from_alpha(const float* alpha, vs_tf_params* out) {
  if (!alpha || !out) return fail_arg("null pointer");
  memset(out, 0, sizeof *out);
  int prev = alpha[0] > 0.0f;
  int nflip = 0;
  out->start = prev;
  for (int b = 0; b < 256; ++b) {
    int v = alpha[b] > 0.0f;
    if (v) {
      out->vis[b >> 5] |= 1u << (b & 31);
      out->nvisible++;
    }
    if (b > 0 && v != prev) {
      if (nflip < 2) out->bound[nflip] = b;
      nflip++;
    }
    prev = v;
  }
  out->mode = nflip == 0 ? 3 : (nflip <= 2 ? nflip : 0);
  return 0;
}

int vs_quantize_f32(const float* field, int64_t n, uint8_t* bins, vs_stream_t st) {
  if (n < 0 || (n && (!field || !bins))) return fail_arg("vs_quantize_f32");
  if (n == 0) return 0;
  k_quantize<<<(unsigned)cdiv(n, 256), 256, 0, S(st)>>>(field, n, bins);
  return check_launch("k_quantize");
}

int vs_classify_summary(const uint8_t* bins, int nx, int ny, int nz, const vs_tf_params* tf,
                        uint32_t* summary, uint32_t* bits, unsigned long long* count,
                        vs_stream_t st) {
  if (!bins || !tf || !summary || nx < 1 || ny < 1 || nz < 1)
    return fail_arg("vs_classify_summary");
  if (nz % 16 != 0) return fail_arg("vs_classify_summary needs nz % 16 == 0");
  if ((uintptr_t)bins & 15) return fail_arg("vs_classify_summary needs 16-byte aligned bins");
  const int nbx = (int)cdiv(nx, 8), nby = (int)cdiv(ny, 8), nbz = (int)cdiv(nz, 8);
  const int nzc = (int)cdiv(nz, 512);
  const int64_t ntasks = (int64_t)nbx * nby * nzc;
  const unsigned grid = (unsigned)cdiv(ntasks, SUMMARY_WARPS);
  if (bits && count)
    k_brick_summary_out<true, true><<<grid, SUMMARY_WARPS * 32, 0, S(st)>>>(
        bins, nx, ny, nz, tf, summary, bits, count, nbx, nby, nbz, nzc, ntasks);
  else if (bits)
    k_brick_summary_out<true, false><<<grid, SUMMARY_WARPS * 32, 0, S(st)>>>(
        bins, nx, ny, nz, tf, summary, bits, count, nbx, nby, nbz, nzc, ntasks);
  else if (count)
    k_brick_summary_out<false, true><<<grid, SUMMARY_WARPS * 32, 0, S(st)>>>(
        bins, nx, ny, nz, tf, summary, bits, count, nbx, nby, nbz, nzc, ntasks);
  else
    k_brick_summary<<<grid, SUMMARY_WARPS * 32, 0, S(st)>>>(bins, nx, ny, nz, tf, summary,
                                                            nbx, nby, nbz, nzc, ntasks);
  return check_launch("k_brick_summary");
}

int vs_classify_bits(const uint8_t* bins, int nx, int ny, int nz, const vs_tf_params* tf,
                     uint32_t* bits, unsigned long long* count, vs_stream_t st) {
  if (!bins || !tf || !bits || nx < 1 || ny < 1 || nz < 1) return fail_arg("vs_classify_bits");
  if (nz % 32 == 0 && nz <= 1024 && (reinterpret_cast<uintptr_t>(bins) & 15) == 0) {
    dim3 grid((unsigned)cdiv(ny, 32), (unsigned)cdiv(nx, CP_XC));
    k_classify_pack<false><<<grid, 1024, 0, S(st)>>>(bins, nx, ny, nz, tf, bits, count, nullptr);
    return check_launch("k_classify_pack");
  }
  const int64_t nwords = (int64_t)nx * ny * nzw_of(nz);
  k_classify_bits<<<(unsigned)cdiv(nwords, 256), 256, 0, S(st)>>>(bins, nx, ny, nz, tf, bits,
                                                                    count);
  return check_launch("k_classify_bits");
}

int vs_classify_dilate_bits_bbox(const uint8_t* bins, int nx, int ny, int nz,
                                 const vs_tf_params* tf, uint32_t* bits,
                                 unsigned long long* count, int* bbox, vs_stream_t st) {
  if (!bins || !tf || !bits || nx < 1 || ny < 1 || nz < 1)
    return fail_arg("vs_classify_dilate_bits");
  if (nz % 32 != 0 || nz > 1024 || (reinterpret_cast<uintptr_t>(bins) & 15) != 0)
    return fail_arg("vs_classify_dilate_bits: needs nz % 32 == 0, nz <= 1024, 16-byte aligned");
  if (bbox) {
    k_bbox_init<<<1, 32, 0, S(st)>>>(bbox);
    VS_TRY(check_launch("k_bbox_init"));
  }
  dim3 grid((unsigned)cdiv(ny, CP_TY), (unsigned)cdiv(nx, CP_XC));
  const size_t smem = VS_CP_BULK ? 128 + (size_t)CP_NS * (CP_TY + 2) * nz : 0;
  if (smem > 48 * 1024)
    VS_CUDA(cudaFuncSetAttribute(k_classify_pack<true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "k_classify_pack smem");
  k_classify_pack<true><<<grid, 32 * (CP_TY + 2), smem, S(st)>>>(bins, nx, ny, nz, tf, bits,
                                                                count, bbox);
  return check_launch("k_classify_pack<dilate>");
}

int vs_classify_dilate_bits(const uint8_t* bins, int nx, int ny, int nz, const vs_tf_params* tf,
                            uint32_t* bits, unsigned long long* count, vs_stream_t st) {
  return vs_classify_dilate_bits_bbox(bins, nx, ny, nz, tf, bits, count, nullptr, st);
}

int vs_dilate_bits(const uint32_t* in, int nx, int ny, int nz, uint32_t* out, vs_stream_t st) {
  if (!in || !out || in == out || nx < 1 || ny < 1 || nz < 1) return fail_arg("vs_dilate_bits");
  if (ny > 65535) return fail_arg("vs_dilate_bits: ny > 65535");
  const int nzw = (int)nzw_of(nz);
  const int bx = nzw >= 128 ? 128 : 32;
  dim3 grid((unsigned)cdiv(nzw, bx), (unsigned)ny, (unsigned)cdiv(nx, DIL_XCHUNK));
  k_dilate<<<grid, bx, 0, S(st)>>>(in, nx, ny, nz, out);
  return check_launch("k_dilate");
}

int vs_pack_bits(const uint8_t* bools, int nx, int ny, int nz, uint32_t* bits, vs_stream_t st) {
  if (!bools || !bits || nx < 1 || ny < 1 || nz < 1) return fail_arg("vs_pack_bits");
  const int64_t nrows = (int64_t)nx * ny;
  k_pack<<<(unsigned)cdiv(nrows * nzw_of(nz), 256), 256, 0, S(st)>>>(bools, nrows, nz, bits);
  return check_launch("k_pack");
}

int vs_unpack_bits(const uint32_t* bits, int nx, int ny, int nz, uint8_t* bools,
                   vs_stream_t st) {
  if (!bools || !bits || nx < 1 || ny < 1 || nz < 1) return fail_arg("vs_unpack_bits");
  const int64_t nrows = (int64_t)nx * ny;
  k_unpack<<<(unsigned)cdiv(nrows * nz, 256), 256, 0, S(st)>>>(bits, nrows, nz, bools);
  return check_launch("k_unpack");
}

int vs_count_bits(const uint32_t* bits, int nx, int ny, int nz, unsigned long long* count,
                  vs_stream_t st) {
  if (!bits || !count || nx < 1 || ny < 1 || nz < 1) return fail_arg("vs_count_bits");
  const int64_t nwords = (int64_t)nx * ny * nzw_of(nz);
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(nwords, 256), 148 * 16);
  k_count_bits<<<grid, 256, 0, S(st)>>>(bits, nwords, count);
  return check_launch("k_count_bits");
}

int vs_vote_cells(const uint32_t* bits, int nx, int ny, int nz, int cs, uint8_t* flags,
                  vs_stream_t st) {
  if (!bits || !flags || nx < 1 || ny < 1 || nz < 1 || cs < 1) return fail_arg("vs_vote_cells");
  const int ncx = (int)cdiv(nx, cs), ncy = (int)cdiv(ny, cs), ncz = (int)cdiv(nz, cs);
  const int64_t n = (int64_t)ncx * ncy * ncz;
  if (cs == 16 && nz % 32 == 0 && nz <= 1024 && (reinterpret_cast<uintptr_t>(bits) & 15) == 0 &&
      (nz / 32) % 4 == 0) {
    k_vote_cells16<<<(unsigned)(ncx * ncy), 256, 0, S(st)>>>(bits, nx, ny, nz, ncy, ncz, flags);
    return check_launch("k_vote_cells16");
  }
  k_vote_cells<<<(unsigned)cdiv(n, 128), 128, 0, S(st)>>>(bits, nx, ny, nz, cs, ncx, ncy, ncz,
                                                          flags);
  return check_launch("k_vote_cells");
}

int vs_morton_side(int nbx, int nby, int nbz) {
  int m = std::max(nbx, std::max(nby, nbz));
  if (m > 1024 || m < 1) return VS_ERANGE;
  int p = 8;
  while (p < m) p <<= 1;
  return p;
}

static int flags_tiles(int mode, const uint32_t* src, const uint32_t* const* chans,
                       const int32_t* tf_params, int nch,
                       int nx, int ny, int nz, int P, uint32_t* bitmap, uint32_t* tile_counts,
                       uint8_t* cell16, uint32_t* grid, cudaStream_t st) {
  const int nbx = (int)cdiv(nx, 8), nby = (int)cdiv(ny, 8), nbz = (int)cdiv(nz, 8);
  if (P != vs_morton_side(nbx, nby, nbz)) return fail_arg("flags to bitmap: P");
  const int64_t ntiles = (int64_t)P * P * P / 512;
  const int ncx = (int)cdiv(nx, 16), ncy = (int)cdiv(ny, 16), ncz = (int)cdiv(nz, 16);
  const int64_t nb = (int64_t)nbx * nby * nbz;
  if (grid && (nbz & 7) != 0)  // bits set by atomics
    VS_CUDA(cudaMemsetAsync(grid, 0, ((nb + 31) / 32) * 4, st), "memset brick grid");
  else if (grid && (nb & 31) != 0)  // padding bits of the last word (never stored by bytes)
    VS_CUDA(cudaMemsetAsync(grid + nb / 32, 0, 4, st), "memset brick grid tail");
  if (mode == FL_PRESENCE && !cell16 && (nbz & 31) == 0 && (int64_t)nbx * nby <= 65535) {
    VS_CUDA(cudaMemsetAsync(bitmap, 0, ntiles * 16 * 4, st), "memset bitmap");
    VS_CUDA(cudaMemsetAsync(tile_counts, 0, ntiles * 4, st), "memset tile counts");
    const int bt = nbz >= 256 ? 256 : nbz;
    k_presence_vote<<<dim3((unsigned)cdiv(nbz, bt), (unsigned)(nbx * nby)), bt, 0, st>>>(
        chans, tf_params, nch, nby, nbz, bitmap, tile_counts, grid);
    return check_launch("k_presence_vote");
  }
  const unsigned g = (unsigned)std::min<int64_t>(ntiles, (int64_t)sm_count() * 8);
  if (mode == FL_SUMMARY_DILATE)
    k_flags_tiles<FL_SUMMARY_DILATE><<<g, FL_T, 0, st>>>(src, chans, tf_params, nch, nbx, nby, nbz,
                                                        ntiles, bitmap, tile_counts, cell16, ncx,
                                                        ncy, ncz, grid);
  else if (mode == FL_SUMMARY)
    k_flags_tiles<FL_SUMMARY><<<g, FL_T, 0, st>>>(src, chans, tf_params, nch, nbx, nby, nbz, ntiles,
                                                 bitmap, tile_counts, cell16, ncx, ncy, ncz,
                                                 grid);
  else
    k_flags_tiles<FL_PRESENCE><<<g, FL_T, 0, st>>>(src, chans, tf_params, nch, nbx, nby, nbz, ntiles,
                                                  bitmap, tile_counts, cell16, ncx, ncy, ncz,
                                                  grid);
  return check_launch("k_flags_tiles");
}

int vs_summary_to_bitmap(const uint32_t* summary, int nx, int ny, int nz, int dilate, int P,
                         uint32_t* bitmap, uint32_t* tile_counts, uint8_t* cell16,
                         uint32_t* grid, vs_stream_t st) {
  if (!summary || !bitmap || !tile_counts || nx < 1 || ny < 1 || nz < 1)
    return fail_arg("vs_summary_to_bitmap");
  return flags_tiles(dilate ? FL_SUMMARY_DILATE : FL_SUMMARY, summary, nullptr, nullptr, 1, nx,
                     ny, nz, P,
                     bitmap, tile_counts, cell16, grid, S(st));
}

int64_t vs_presence_words(int nx, int ny, int nz) {
  if (nx < 1 || ny < 1 || nz < 1) return -1;
  return cdiv(nx, 8) * cdiv(ny, 8) * cdiv(nz, 8) * 8;
}

int vs_presence_build_slab(const uint8_t* bins, int nx, int ny, int nz, int bx0, int bx1,
                           uint32_t* presence, vs_stream_t st) {
  if (!bins || !presence || nx < 1 || ny < 1 || nz < 1 || nz % 16 != 0 ||
      ((uintptr_t)bins & 15) != 0)
    return fail_arg("vs_presence_build (needs nz % 16 == 0, 16-byte aligned bins)");
  const int nbx = (int)cdiv(nx, 8), nby = (int)cdiv(ny, 8), nbz = (int)cdiv(nz, 8);
  if (bx0 < 0 || bx1 > nbx || bx0 > bx1)
    return fail_arg("vs_presence_build_slab: brick slab range outside [0, nbx]");
  if (bx0 == bx1) return 0;
  const size_t smem = (size_t)nbz * 8 * 4;
  if (smem > 48 * 1024)
    VS_CUDA(cudaFuncSetAttribute(k_presence, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem), "presence smem");
  k_presence<<<(unsigned)((int64_t)(bx1 - bx0) * nby), PR_T, smem, S(st)>>>(
      bins, nx, ny, nz, nby, nbz, bx0, presence);
  return check_launch("k_presence");
}

int vs_presence_build(const uint8_t* bins, int nx, int ny, int nz, uint32_t* presence,
                      vs_stream_t st) {
  return vs_presence_build_slab(bins, nx, ny, nz, 0, nx < 1 ? 0 : (int)cdiv(nx, 8), presence,
                                st);
}

int vs_presence_to_bitmap(const uint32_t* const* presence, const int32_t* tf_params, int nch,
                          int nx, int ny, int nz, int P, uint32_t* bitmap,
                          uint32_t* tile_counts, uint8_t* cell16, uint32_t* grid,
                          vs_stream_t st) {
  if (!presence || !tf_params || !bitmap || !tile_counts || nch < 1 || nch > 4 || nx < 1 ||
      ny < 1 || nz < 1)
    return fail_arg("vs_presence_to_bitmap");
  return flags_tiles(FL_PRESENCE, nullptr, presence, tf_params, nch, nx, ny, nz, P, bitmap,
                     tile_counts, cell16, grid, S(st));
}

int vs_flags_to_bitmap(const uint8_t* flags, int nbx, int nby, int nbz, int P, uint32_t* bitmap,
                       uint32_t* tile_counts, vs_stream_t st) {
  if (!flags || !bitmap || !tile_counts || nbx < 1 || nby < 1 || nbz < 1)
    return fail_arg("vs_flags_to_bitmap");
  if (P != vs_morton_side(nbx, nby, nbz)) return fail_arg("vs_flags_to_bitmap: P");
  const int64_t nwords = (int64_t)P * P * P / 32;
  const int64_t ntiles = nwords / 16;
  VS_CUDA(cudaMemsetAsync(bitmap, 0, nwords * 4, S(st)), "memset bitmap");
  const int64_t n = (int64_t)nbx * nby * nbz;
  k_flags_scatter<<<(unsigned)cdiv(n, 256), 256, 0, S(st)>>>(flags, nbx, nby, nbz, bitmap);
  VS_TRY(check_launch("k_flags_scatter"));
  k_tile_counts<<<(unsigned)cdiv(ntiles, 256), 256, 0, S(st)>>>(bitmap, ntiles, tile_counts);
  return check_launch("k_tile_counts");
}

size_t vs_bricks_workspace(int nbx, int nby, int nbz) {
  const int64_t n = (int64_t)nbx * nby * nbz;
  size_t cub_bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, cub_bytes, thrust::counting_iterator<int64_t>(0),
                             (const uint8_t*)nullptr, (int64_t*)nullptr, (int*)nullptr, (int)n);
  Bump b(nullptr);
  b.take<uint8_t>(n);
  b.take<int64_t>(n);
  b.take<char>(cub_bytes);
  return b.off + 256;
}

int vs_bricks_from_bitmap(const uint32_t* bitmap, int nbx, int nby, int nbz, int P,
                          int32_t* coords, uint32_t* codes, int* n_out, void* ws,
                          size_t ws_bytes, vs_stream_t st) {
  if (!bitmap || !coords || !codes || !n_out || nbx < 1 || nby < 1 || nbz < 1)
    return fail_arg("vs_bricks_from_bitmap");
  if (ws_bytes < vs_bricks_workspace(nbx, nby, nbz)) return VS_EWORKSPACE;
  const int64_t n = (int64_t)nbx * nby * nbz;
  size_t cub_bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, cub_bytes, thrust::counting_iterator<int64_t>(0),
                             (const uint8_t*)nullptr, (int64_t*)nullptr, (int*)nullptr, (int)n);
  Bump b(ws);
  uint8_t* flags = b.take<uint8_t>(n);
  int64_t* idx = b.take<int64_t>(n);
  void* tmp = b.take<char>(cub_bytes);
  k_bitmap_to_scan_flags<<<(unsigned)cdiv(n, 256), 256, 0, S(st)>>>(bitmap, nbx, nby, nbz,
                                                                    flags);
  VS_TRY(check_launch("k_bitmap_to_scan_flags"));
  VS_CUDA(cub::DeviceSelect::Flagged(tmp, cub_bytes, thrust::counting_iterator<int64_t>(0),
                                     flags, idx, n_out, (int)n, S(st)),
          "DeviceSelect::Flagged");
  k_decode_scan<<<(unsigned)cdiv(n, 256), 256, 0, S(st)>>>(idx, n_out, nby, nbz, coords, codes,
                                                           n);
  return check_launch("k_decode_scan");
}

}  // extern "C"
