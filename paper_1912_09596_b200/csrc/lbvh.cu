// LBVH construction over non-empty bricks: build_lbvh (lbvh.py:216-264).
//
//   bitmap path (bricks from flag_bricks): the Morton bitmap already IS the sorted order, so
//     k_leaves_from_bitmap ranks each set bit (tile offsets from one exclusive scan) and
//     emits the leaf rows; no sort is needed because brick codes are distinct and the
//     reference's stable argsort of (code << 32 | scan index) then orders by code alone.
//   bricks path (an arbitrary BrickSet, codes may repeat): keys = code << 32 | index,
//     CUB radix sort (equals numpy's stable argsort on unique 64-bit keys), leaf rows.
//   both: k_karras (lbvh.py:167-200, one thread per internal node, 64-bit keys so equal codes
//     break ties on the index exactly like _common_prefix lbvh.py:153-164), then k_refit
//     (lbvh.py:203-213): bottom-up unions with per-node arrival counters; min/max is
//     order-independent, so the boxes equal the reference's children-before-parents sweep.
//     The same pass yields height() (lbvh.py:128-144) as the root's subtree height.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace vs {

// δ(i, j) of lbvh.py:153-164: leading zeros of keys[i] ^ keys[j]; -1 outside [0, n).
__device__ __forceinline__ int delta(const uint64_t* __restrict__ k, int64_t i, int64_t j,
                                     int64_t n) {
  if (j < 0 || j >= n) return -1;
  uint64_t x = k[i] ^ k[j];
  return x == 0 ? 64 : __clzll((long long)x);
}

// Thread per 32-code bitmap word: rank = tile offset + popcounts of the earlier words of the
// tile (16-lane segmented warp scan) + bits below in the word; each set bit emits its leaf.
__global__ void k_leaves_from_bitmap(const uint32_t* __restrict__ bitmap,
                                     const uint32_t* __restrict__ tile_off, int bs, int nx,
                                     int ny, int nz, int64_t ntiles, uint64_t* __restrict__ keys,
                                     int32_t* __restrict__ lo, int32_t* __restrict__ hi,
                                     int32_t* __restrict__ left, int32_t* __restrict__ right,
                                     int32_t* __restrict__ leaf_brick,
                                     int32_t* __restrict__ brick_coords, int* __restrict__ info) {
  const int64_t wi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // word index
  const int64_t nwords = ntiles * 16;
  const int64_t n = tile_off[ntiles];
  if (wi == 0) info[0] = (int)n;
  uint32_t word = wi < nwords ? __ldg(bitmap + wi) : 0u;
  const uint32_t c = __popc(word);
  uint32_t incl = c;
  const int seg = threadIdx.x & 15;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o, 16);
    if (seg >= o) incl += u;
  }
  if (wi >= nwords || !word) return;
  int64_t p = (int64_t)tile_off[wi >> 4] + (incl - c);
  while (word) {
    const int bit = __ffs(word) - 1;
    word &= word - 1;
    const uint32_t code = (uint32_t)(wi * 32 + bit);
    const int bx = (int)compact10(code), by = (int)compact10(code >> 1),
              bz = (int)compact10(code >> 2);
    keys[p] = (uint64_t)code << 32;  // low word irrelevant: codes are distinct
    brick_coords[3 * p] = bx;
    brick_coords[3 * p + 1] = by;
    brick_coords[3 * p + 2] = bz;
    const int64_t row = n - 1 + p;
    lo[3 * row] = bx * bs;
    lo[3 * row + 1] = by * bs;
    lo[3 * row + 2] = bz * bs;
    hi[3 * row] = min(bx * bs + bs, nx);
    hi[3 * row + 1] = min(by * bs + bs, ny);
    hi[3 * row + 2] = min(bz * bs + bs, nz);
    left[row] = -1;
    right[row] = -1;
    leaf_brick[row] = (int32_t)p;
    ++p;
  }
}

__global__ void k_make_keys(const uint32_t* __restrict__ codes, int64_t n,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((uint64_t)codes[i] << 32) | (uint64_t)i;
  vals[i] = (int32_t)i;
}

__global__ void k_leaves_from_sorted(const int32_t* __restrict__ coords,
                                     const int32_t* __restrict__ order, int64_t n, int bs,
                                     int nx, int ny, int nz, int32_t* __restrict__ lo,
                                     int32_t* __restrict__ hi, int32_t* __restrict__ left,
                                     int32_t* __restrict__ right,
                                     int32_t* __restrict__ leaf_brick,
                                     int32_t* __restrict__ brick_coords, int* __restrict__ info) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) info[0] = (int)n;
  if (p >= n) return;
  const int64_t src = order[p];
  const int bx = coords[3 * src], by = coords[3 * src + 1], bz = coords[3 * src + 2];
  brick_coords[3 * p] = bx;
  brick_coords[3 * p + 1] = by;
  brick_coords[3 * p + 2] = bz;
  const int64_t row = n - 1 + p;
  // lbvh.py:231-232: leaf_lo = coords*bs (int64), leaf_hi = min(leaf_lo + bs, dims)
  const int64_t l0 = (int64_t)bx * bs, l1 = (int64_t)by * bs, l2 = (int64_t)bz * bs;
  lo[3 * row] = (int32_t)l0;
  lo[3 * row + 1] = (int32_t)l1;
  lo[3 * row + 2] = (int32_t)l2;
  hi[3 * row] = (int32_t)(l0 + bs < nx ? l0 + bs : (int64_t)nx);
  hi[3 * row + 1] = (int32_t)(l1 + bs < ny ? l1 + bs : (int64_t)ny);
  hi[3 * row + 2] = (int32_t)(l2 + bs < nz ? l2 + bs : (int64_t)nz);
  left[row] = -1;
  right[row] = -1;
  leaf_brick[row] = (int32_t)p;
}

// Karras 2012 over sorted keys; n read from info[0] (device) so the launch needs no host sync.
__global__ void k_karras(const uint64_t* __restrict__ keys, const int* __restrict__ info,
                         int64_t cap, int32_t* __restrict__ left, int32_t* __restrict__ right,
                         int32_t* __restrict__ leaf_brick, int32_t* __restrict__ parent,
                         int2* __restrict__ range) {
  const int64_t n = info[0];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && n >= 1) parent[0] = -1;  // root (the single leaf when n == 1)
  if (i >= n - 1) return;
  const int d = delta(keys, i, i + 1, n) > delta(keys, i, i - 1, n) ? 1 : -1;
  const int dmin = delta(keys, i, i - d, n);
  int64_t lmax = 2;
  while (delta(keys, i, i + lmax * d, n) > dmin) lmax *= 2;
  int64_t l = 0;
  for (int64_t t = lmax / 2; t >= 1; t /= 2)
    if (delta(keys, i, i + (l + t) * d, n) > dmin) l += t;
  const int64_t j = i + l * d;
  const int dnode = delta(keys, i, j, n);
  int64_t s = 0, t = l;
  while (true) {
    t = (t + 1) / 2;
    if (delta(keys, i, i + (s + t) * d, n) > dnode) s += t;
    if (t == 1) break;
  }
  const int64_t gamma = i + s * d + min(d, 0);
  const int64_t lo_i = min(i, j), hi_i = max(i, j);
  const int64_t lc = (lo_i == gamma) ? (n - 1) + gamma : gamma;
  const int64_t rc = (hi_i == gamma + 1) ? (n - 1) + gamma + 1 : gamma + 1;
  left[i] = (int32_t)lc;
  right[i] = (int32_t)rc;
  leaf_brick[i] = -1;
  range[i] = make_int2((int)lo_i, (int)hi_i);
  parent[lc] = (int32_t)i;
  parent[rc] = (int32_t)i;
}

// Bottom-up refit: thread per leaf; the second arrival at a node unions both children.
__global__ void k_refit(int32_t* __restrict__ lo,
                        int32_t* __restrict__ hi, const int32_t* __restrict__ left,
                        const int32_t* __restrict__ right, const int32_t* __restrict__ parent,
                        int32_t* __restrict__ visit, int32_t* __restrict__ hgt,
                        int* info) {
  const int64_t n = info[0];
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) {
    if (n == 0) info[1] = 0;
    if (n == 1) info[1] = 1;
  }
  if (n < 2 || p >= n) return;
  int64_t node = parent[n - 1 + p];
  while (node >= 0) {
    __threadfence();
    if (atomicAdd(&visit[node], 1) == 0) return;
    __threadfence();
    const int32_t l = __ldcg(left + node), r = __ldcg(right + node);
    int32_t b[6];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      b[a] = min(__ldcg(lo + 3 * l + a), __ldcg(lo + 3 * r + a));
      b[3 + a] = max(__ldcg(hi + 3 * l + a), __ldcg(hi + 3 * r + a));
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      __stcg(lo + 3 * node + a, b[a]);
      __stcg(hi + 3 * node + a, b[3 + a]);
    }
    const int hl = (l >= n - 1) ? 1 : __ldcg(hgt + l);
    const int hr = (r >= n - 1) ? 1 : __ldcg(hgt + r);
    const int h = 1 + max(hl, hr);
    __stcg(hgt + node, h);
    if (node == 0) {
      info[1] = h;
      return;
    }
    node = __ldcg(parent + node);
  }
}

static size_t scan_temp_bytes(int64_t items) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)items);
  return b;
}

static size_t sort_temp_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return b;
}

// Refit with the lower levels in shared memory: a CTA owns RC consecutive leaves; every
// internal node whose leaf range lies inside the CTA's chunk is refit with shared-memory
// arrival counters (no global fences), and only the nodes whose range crosses chunks -- about
// log2(n / RC) levels -- climb with the global protocol.  Unions are order-independent, so the
// boxes and heights equal k_refit's (and the reference's sweep).
constexpr int RC = 1024;

__global__ void __launch_bounds__(RC)
    k_refit_chunked(int32_t* __restrict__ lo, int32_t* __restrict__ hi,
                    const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                    const int32_t* __restrict__ parent, const int2* __restrict__ range,
                    int32_t* __restrict__ visit, int32_t* __restrict__ hgt, int* info) {
  __shared__ int s_box[RC][6];
  __shared__ int s_cnt[RC];
  __shared__ int s_h[RC];
  const int64_t n = info[0];
  const int t = threadIdx.x;
  if (blockIdx.x == 0 && t == 0) {
    if (n == 0) info[1] = 0;
    if (n == 1) info[1] = 1;
  }
  if (n < 2) return;
  const int64_t c0 = (int64_t)blockIdx.x * RC;
  if (c0 >= n) return;
  const int64_t c1 = c0 + RC < n ? c0 + RC : n;
  s_cnt[t] = 0;
  __syncthreads();
  const int64_t p = c0 + t;
  if (p >= c1) return;
  int64_t node = parent[n - 1 + p];
  while (node >= 0) {
    const int2 rg = range[node];
    const int32_t l = left[node], r = right[node];
    int b[6], hl, hr;
    if (rg.x >= c0 && rg.y < c1) {  // inside the chunk: shared-memory protocol
      __threadfence_block();
      if (atomicAdd(&s_cnt[node - c0], 1) == 0) return;
      __threadfence_block();
      int bl[6], br[6];
      if (l >= n - 1) {
        for (int a = 0; a < 3; ++a) { bl[a] = lo[3 * l + a]; bl[3 + a] = hi[3 * l + a]; }
        hl = 1;
      } else {
        for (int a = 0; a < 6; ++a) bl[a] = s_box[l - c0][a];
        hl = s_h[l - c0];
      }
      if (r >= n - 1) {
        for (int a = 0; a < 3; ++a) { br[a] = lo[3 * r + a]; br[3 + a] = hi[3 * r + a]; }
        hr = 1;
      } else {
        for (int a = 0; a < 6; ++a) br[a] = s_box[r - c0][a];
        hr = s_h[r - c0];
      }
      for (int a = 0; a < 3; ++a) {
        b[a] = min(bl[a], br[a]);
        b[3 + a] = max(bl[3 + a], br[3 + a]);
      }
      const int h = 1 + max(hl, hr);
      for (int a = 0; a < 6; ++a) s_box[node - c0][a] = b[a];
      s_h[node - c0] = h;
      for (int a = 0; a < 3; ++a) { lo[3 * node + a] = b[a]; hi[3 * node + a] = b[3 + a]; }
      hgt[node] = h;
      if (node == 0) { info[1] = h; return; }
    } else {  // crossing chunks: global protocol
      __threadfence();
      if (atomicAdd(&visit[node], 1) == 0) return;
      __threadfence();
      for (int a = 0; a < 3; ++a) {
        b[a] = min(__ldcg(lo + 3 * l + a), __ldcg(lo + 3 * r + a));
        b[3 + a] = max(__ldcg(hi + 3 * l + a), __ldcg(hi + 3 * r + a));
      }
      hl = (l >= n - 1) ? 1 : __ldcg(hgt + l);
      hr = (r >= n - 1) ? 1 : __ldcg(hgt + r);
      const int h = 1 + max(hl, hr);
      for (int a = 0; a < 3; ++a) {
        __stcg(lo + 3 * node + a, b[a]);
        __stcg(hi + 3 * node + a, b[3 + a]);
      }
      __stcg(hgt + node, h);
      if (node == 0) { info[1] = h; return; }
    }
    node = parent[node];
  }
}

// ---- bitmap path: sort-free leaves, Karras emission and range-reduction boxes ---------------
// The leaves of the bitmap path are the set bits in code order, so every internal node's box is
// the union of a CONTIGUOUS run of leaf boxes -- its Karras range [a, b] (lbvh.py:167-200; the
// refit of lbvh.py:203-213 unions exactly the leaves of the subtree).  Boxes are therefore
// computed as range reductions instead of a bottom-up climb: a CTA owns TC consecutive leaves
// and the TC internal nodes with the same indices (node i always has i as one end of its range);
// a node whose range lies inside the chunk reduces from shared-memory warp prefix / suffix boxes
// and block totals, and the few nodes whose range crosses a chunk boundary are finished by a
// second kernel from per-leaf chunk prefix / suffix boxes and the chunk totals.  Brick
// coordinates are < 1024, so a box is kept as packed 16-bit (x | y << 16, z) minima / maxima.
constexpr int TC = 512;

__device__ __forceinline__ uint4 box_empty() { return make_uint4(~0u, ~0u, 0u, 0u); }
__device__ __forceinline__ uint4 box_union(uint4 a, uint4 b) {
  return make_uint4(__vminu2(a.x, b.x), min(a.y, b.y), __vmaxu2(a.z, b.z), max(a.w, b.w));
}
__device__ __forceinline__ uint4 shfl_box(uint4 v, int d, bool up) {
  uint4 r;
  if (up) {
    r.x = __shfl_up_sync(0xffffffffu, v.x, d); r.y = __shfl_up_sync(0xffffffffu, v.y, d);
    r.z = __shfl_up_sync(0xffffffffu, v.z, d); r.w = __shfl_up_sync(0xffffffffu, v.w, d);
  } else {
    r.x = __shfl_down_sync(0xffffffffu, v.x, d); r.y = __shfl_down_sync(0xffffffffu, v.y, d);
    r.z = __shfl_down_sync(0xffffffffu, v.z, d); r.w = __shfl_down_sync(0xffffffffu, v.w, d);
  }
  return r;
}
// voxel box of a brick-coordinate box: lo = c*bs, hi = min(c*bs + bs, dims) (lbvh.py:231-232;
// the union of clipped leaf boxes is the clipped box of the extreme bricks)
__device__ __forceinline__ void store_box(uint4 b, int bs, int nx, int ny, int nz, int64_t row,
                                          int32_t* __restrict__ lo, int32_t* __restrict__ hi) {
  lo[3 * row] = (int)(b.x & 0xffffu) * bs;
  lo[3 * row + 1] = (int)(b.x >> 16) * bs;
  lo[3 * row + 2] = (int)b.y * bs;
  hi[3 * row] = min((int)(b.z & 0xffffu) * bs + bs, nx);
  hi[3 * row + 1] = min((int)(b.z >> 16) * bs + bs, ny);
  hi[3 * row + 2] = min((int)b.w * bs + bs, nz);
}

// Exclusive scan of the tile popcounts in one CTA (off[ntiles] = n), for ntiles <= 1024 * 32:
// all loads issued up front (coalesced, strided by the CTA width), then one block scan per
// 1024-entry round with a running carry.
constexpr int SCAN_T = 1024, SCAN_PER = 32;
__global__ void __launch_bounds__(SCAN_T)
    k_tile_scan(const uint32_t* __restrict__ cnt, int64_t ntiles, uint32_t* __restrict__ off) {
  __shared__ uint32_t ws[2][32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int rounds = (int)((ntiles + SCAN_T - 1) / SCAN_T);
  uint32_t v[SCAN_PER];
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    const int64_t i = (int64_t)k * SCAN_T + t;
    v[k] = (k < rounds && i < ntiles) ? __ldg(cnt + i) : 0u;
  }
  uint32_t carry = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    if (k < rounds) {  // uniform
      uint32_t incl = v[k];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) ws[k & 1][warp] = incl;
      __syncthreads();
      uint32_t w = ws[k & 1][lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += u;
      }
      const uint32_t before = __shfl_sync(0xffffffffu, wi - w, warp);
      const uint32_t total = __shfl_sync(0xffffffffu, wi, 31);
      const int64_t i = (int64_t)k * SCAN_T + t;
      if (i < ntiles) off[i] = carry + before + incl - v[k];
      carry += total;
    }
  }
  if (t == 0) off[ntiles] = carry;
}

// Sampled codes for the Karras searches: every S-th sorted code (S = 2^slog >= 64 so that at most
// NSAMP samples exist), written by k_leaves_coop and staged in shared memory by k_tree_chunk.
constexpr int NSAMP = 4096;
__device__ __forceinline__ int samp_log(int64_t n) {
  int lg = 6;
  while (((n + (1LL << lg) - 1) >> lg) > NSAMP) ++lg;
  return lg;
}

// Leaves: warp per two 512-code tiles (lane = bitmap word); the warp's leaves are one
// contiguous run of ranks, staged in shared memory and written row-coalesced.  Also the
// renderer's C-order leaf-brick bit grid (optional, pre-zeroed) and info {n, height sentinel}.
constexpr int LV_WARPS = 8;
__global__ void __launch_bounds__(LV_WARPS * 32)
    k_leaves_coop(const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ off, int bs,
                  int nx, int ny, int nz, int nby, int nbz, int64_t ntiles,
                  uint32_t* __restrict__ codes, int32_t* __restrict__ lo,
                  int32_t* __restrict__ hi, int32_t* __restrict__ left,
                  int32_t* __restrict__ right, int32_t* __restrict__ leaf_brick,
                  int32_t* __restrict__ brick_coords, uint32_t* __restrict__ grid,
                  int* __restrict__ info, int* __restrict__ cross_count,
                  uint32_t* __restrict__ samp) {
  __shared__ uint32_t stage[LV_WARPS][1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = off[ntiles];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = (int)n;
    info[1] = n == 0 ? 0 : (n == 1 ? 1 : -1);  // -1: height computed on demand
    *cross_count = 0;
  }
  const int64_t pair = (int64_t)blockIdx.x * LV_WARPS + warp;
  const int64_t t0 = 2 * pair;
  if (t0 >= ntiles) return;
  const int64_t wi = t0 * 16 + lane;
  const bool valid = t0 + (lane >> 4) < ntiles;
  uint32_t word = valid ? __ldg(bitmap + wi) : 0u;
  const uint32_t c = __popc(word);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o, 16);
    if ((lane & 15) >= o) incl += u;
  }
  const int64_t P0 = off[t0];
  const int64_t P1 = off[(t0 + 2 < ntiles) ? t0 + 2 : ntiles];
  int pos = (int)((int64_t)off[t0 + (lane >> 4)] - P0) + (int)(incl - c);
  while (word) {
    const int bit = __ffs(word) - 1;
    word &= word - 1;
    stage[warp][pos++] = (uint32_t)(wi * 32 + bit);
  }
  __syncwarp();
  const int cnt = (int)(P1 - P0);
  const int slog = samp_log(n);
  for (int k = lane; k < cnt; k += 32) {
    const uint32_t code = stage[warp][k];
    const int64_t p = P0 + k;
    const int bx = (int)compact10(code), by = (int)compact10(code >> 1),
              bz = (int)compact10(code >> 2);
    codes[p] = code;
    if ((p & ((1LL << slog) - 1)) == 0) samp[p >> slog] = code;
    brick_coords[3 * p] = bx;
    brick_coords[3 * p + 1] = by;
    brick_coords[3 * p + 2] = bz;
    const int64_t row = n - 1 + p;
    lo[3 * row] = bx * bs;
    lo[3 * row + 1] = by * bs;
    lo[3 * row + 2] = bz * bs;
    hi[3 * row] = min(bx * bs + bs, nx);
    hi[3 * row + 1] = min(by * bs + bs, ny);
    hi[3 * row + 2] = min(bz * bs + bs, nz);
    left[row] = -1;
    right[row] = -1;
    leaf_brick[row] = (int32_t)p;
    if (grid) {
      const int64_t lin = ((int64_t)bx * nby + by) * nbz + bz;
      atomicOr(grid + (lin >> 5), 1u << (lin & 31));
    }
  }
}

__device__ __forceinline__ int dlt32(const uint32_t* __restrict__ c, uint32_t ci, int64_t j,
                                     int64_t n) {
  if (j < 0 || j >= n) return -1;
  return __clz(ci ^ __ldg(c + j));  // codes are distinct: never 64 (lbvh.py:153-164)
}
// the same with the codes of [base, base + 2 TC) staged in shared memory (most searches of
// the chunk's nodes stay inside it)
__device__ __forceinline__ int dlt32s(const uint32_t* __restrict__ c, const uint32_t* sc,
                                      int64_t base, uint32_t ci, int64_t j, int64_t n) {
  if (j < 0 || j >= n) return -1;
  const int64_t r = j - base;
  const uint32_t cj = (r >= 0 && r < 2 * TC) ? sc[r] : __ldg(c + j);
  return __clz(ci ^ cj);
}

// The furthest m in [0, M] with clz(ci ^ code[i + m d]) > thr.  The predicate is monotone in m
// (sorted distinct codes share a shorter prefix with code i the further they are), so this is
// the index _build_radix_tree's doubling + bisection searches find (lbvh.py:178-196): here a
// bisection over the shared-memory samples, then one inside an S-wide block (global codes,
// or the chunk's staged window).
__device__ __forceinline__ int64_t furthest(const uint32_t* __restrict__ codes,
                                            const uint32_t* samp, int slog,
                                            const uint32_t* sc, int64_t cbase, uint32_t ci,
                                            int64_t i, int d, int64_t M, int thr) {
  auto code_at = [&](int64_t j) -> uint32_t {
    const int64_t r = j - cbase;
    return (r >= 0 && r < 2 * TC) ? sc[r] : __ldg(codes + j);
  };
  auto P = [&](uint32_t c) { return (int)__clz(ci ^ c) > thr; };
  if (M <= 0) return 0;
  if (d > 0) {
    const int64_t hi = i + M;
    // samples strictly after i and <= hi: largest one with P (P holds on a prefix)
    int64_t k0 = (i >> slog) + 1, k1 = hi >> slog, base = i;
    if (k0 <= k1 && P(samp[k0])) {
      while (k0 < k1) {
        const int64_t mid = (k0 + k1 + 1) >> 1;
        if (P(samp[mid])) k0 = mid; else k1 = mid - 1;
      }
      base = k0 << slog;
    }
    const int64_t bend = base + (1LL << slog) - 1;
    int64_t lo = base, h = hi < bend ? hi : bend;  // P(lo) holds
    while (lo < h) {
      const int64_t mid = (lo + h + 1) >> 1;
      if (P(code_at(mid))) lo = mid; else h = mid - 1;
    }
    return lo - i;
  }
  const int64_t lo_pos = i - M;
  // samples strictly before i and >= lo_pos: smallest one with P (P holds on a suffix)
  int64_t k1 = (i - 1) >> slog, k0 = (lo_pos + (1LL << slog) - 1) >> slog, base = i;
  if (i > 0 && k0 <= k1 && P(samp[k1])) {
    while (k0 < k1) {
      const int64_t mid = (k0 + k1) >> 1;
      if (P(samp[mid])) k1 = mid; else k0 = mid + 1;
    }
    base = k1 << slog;
  }
  const int64_t bbeg = base - (1LL << slog) + 1;
  int64_t lo = lo_pos > bbeg ? lo_pos : bbeg, h = base;  // P(h) holds
  while (lo < h) {
    const int64_t mid = (lo + h) >> 1;
    if (P(code_at(mid))) h = mid; else lo = mid + 1;
  }
  return i - h;
}

// Karras emission (lbvh.py:167-200) for the chunk's internal nodes + in-chunk range boxes.
__global__ void __launch_bounds__(TC)
    k_tree_chunk(const uint32_t* __restrict__ codes, const int* __restrict__ info, int bs,
                 int nx, int ny, int nz, const int32_t* __restrict__ brick_coords,
                 int32_t* __restrict__ lo, int32_t* __restrict__ hi, int32_t* __restrict__ left,
                 int32_t* __restrict__ right, int32_t* __restrict__ leaf_brick,
                 uint4* __restrict__ cpre, uint4* __restrict__ csuf, uint4* __restrict__ ctot,
                 int4* __restrict__ cross, int* __restrict__ cross_count,
                 const uint32_t* __restrict__ samp_g) {
  extern __shared__ uint32_t s_samp[];  // NSAMP sampled codes (dynamic shared memory)
  // s_leaf: leaf boxes; s_sp[L-1][i]: union of leaves [i, i + 2^L) of i's warp block (clipped to
  // the block), L = 1..4, so any in-block range is two lookups; s_tl[L][w]: the same over the
  // warp-block totals (L = 0: the totals)
  __shared__ uint4 s_leaf[TC], s_sp[4][TC];
  __shared__ uint4 s_tl[4][TC / 32], s_bp[TC / 32], s_bs[TC / 32];
  __shared__ uint32_t s_code[2 * TC];
  const int64_t n = info[0];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  constexpr int NW = TC / 32;
  auto in_block = [&](int a, int e) -> uint4 {  // a <= e, same warp block (local indices)
    if (a == e) return s_leaf[a];
    const int L = min(31 - __clz(e - a + 1), 4);
    return box_union(s_sp[L - 1][a], s_sp[L - 1][e - (1 << L) + 1]);
  };
  const int64_t nchunks = (n + TC - 1) / TC;
  const int slog = samp_log(n);
  const int64_t nsamp = (n + (1LL << slog) - 1) >> slog;
  if (blockIdx.x < nchunks)
    for (int k = t; k < nsamp; k += TC) s_samp[k] = __ldg(samp_g + k);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = ch * TC, c1 = (c0 + TC < n) ? c0 + TC : n;
    const int64_t p = c0 + t;
    const int64_t cbase = c0 - TC / 2;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t j = cbase + q * TC + t;
      s_code[q * TC + t] = (j >= 0 && j < n) ? __ldg(codes + j) : 0u;
    }
    uint4 b = box_empty();
    if (p < c1) {
      const uint32_t x = (uint32_t)brick_coords[3 * p], y = (uint32_t)brick_coords[3 * p + 1],
                     z = (uint32_t)brick_coords[3 * p + 2];
      b = make_uint4(x | (y << 16), z, x | (y << 16), z);
    }
    uint4 pre = b, suf = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint4 u = shfl_box(pre, o, true);
      if (lane >= o) pre = box_union(pre, u);
      const uint4 d = shfl_box(suf, o, false);
      if (lane + o < 32) suf = box_union(suf, d);
    }
    s_leaf[t] = b;
    {
      uint4 sp = b;
#pragma unroll
      for (int L = 1; L <= 4; ++L) {
        const uint4 d = shfl_box(sp, 1 << (L - 1), false);
        if (lane + (1 << (L - 1)) < 32) sp = box_union(sp, d);
        s_sp[L - 1][t] = sp;
      }
    }
    if (lane == 31) s_tl[0][warp] = pre;
    __syncthreads();
    if (warp == 0) {  // exclusive block prefix / suffix unions over the NW warp totals
      const uint4 tv = lane < NW ? s_tl[0][lane] : box_empty();
      uint4 bp = tv, bq = tv, sp = tv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint4 u = shfl_box(bp, o, true);
        if (lane >= o) bp = box_union(bp, u);
        const uint4 d = shfl_box(bq, o, false);
        if (lane + o < 32) bq = box_union(bq, d);
      }
#pragma unroll
      for (int L = 1; L <= 3; ++L) {
        const uint4 d = shfl_box(sp, 1 << (L - 1), false);
        if (lane + (1 << (L - 1)) < NW) sp = box_union(sp, d);
        if (lane < NW) s_tl[L][lane] = sp;
      }
      uint4 ex = shfl_box(bp, 1, true), ey = shfl_box(bq, 1, false);
      if (lane == 0) ex = box_empty();
      if (lane == 31) ey = box_empty();
      if (lane < NW) { s_bp[lane] = ex; s_bs[lane] = ey; }
      if (lane == NW - 1) ctot[ch] = bp;  // the chunk's total
    }
    __syncthreads();
    if (p < c1) {  // chunk-level prefix / suffix boxes of leaf p (for crossing ranges)
      cpre[p] = box_union(s_bp[warp], pre);
      csuf[p] = box_union(suf, s_bs[warp]);
    }
    // internal node i = p (lbvh.py:172-200)
    if (p < n - 1) {
      const int64_t i = p;
      const uint32_t ci = s_code[TC / 2 + t];
      const int d = dlt32s(codes, s_code, cbase, ci, i + 1, n) > dlt32s(codes, s_code, cbase, ci, i - 1, n) ? 1 : -1;
      const int dmin = dlt32s(codes, s_code, cbase, ci, i - d, n);
      // the far end j (furthest index with delta > dmin) and the split s (furthest with
      // delta > delta(i, j)): the same indices as the doubling / bisection of lbvh.py:178-196
      const int64_t l = furthest(codes, s_samp, slog, s_code, cbase, ci, i, d,
                                 d > 0 ? n - 1 - i : i, dmin);
      const int64_t j = i + l * d;
      const int dnode = dlt32s(codes, s_code, cbase, ci, j, n);
      const int64_t s = furthest(codes, s_samp, slog, s_code, cbase, ci, i, d, l, dnode);
      const int64_t gamma = i + s * d + min(d, 0);
      const int64_t a = min(i, j), e = max(i, j);
      left[i] = (int32_t)(a == gamma ? (n - 1) + gamma : gamma);
      right[i] = (int32_t)(e == gamma + 1 ? (n - 1) + gamma + 1 : gamma + 1);
      leaf_brick[i] = -1;
      if (a >= c0 && e < c1) {
        const int la = (int)(a - c0), le = (int)(e - c0);
        const int wa = la >> 5, we = le >> 5;
        uint4 acc;
        if (wa == we) {
          acc = in_block(la, le);
        } else {
          acc = box_union(in_block(la, 32 * wa + 31), in_block(32 * we, le));
          if (we - wa >= 2) {  // whole blocks wa+1 .. we-1
            const int u = wa + 1, v = we - 1, L = 31 - __clz(v - u + 1);
            acc = box_union(acc, box_union(s_tl[L][u], s_tl[L][v - (1 << L) + 1]));
          }
        }
        store_box(acc, bs, nx, ny, nz, i, lo, hi);
      } else {
        const unsigned m = __activemask();
        const int leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(cross_count, __popc(m));
        base = __shfl_sync(m, base, leader);
        cross[base + __popc(m & ((1u << lane) - 1u))] = make_int4((int)i, (int)a, (int)e, 0);
      }
    }
    __syncthreads();
  }
}

// Internal nodes whose range crosses a chunk boundary: warp per node, box = chunk suffix of a
// U totals of the chunks in between U chunk prefix of e.
__global__ void __launch_bounds__(256)
    k_tree_cross(const int4* __restrict__ cross, const int* __restrict__ cross_count, int bs,
                 int nx, int ny, int nz, const uint4* __restrict__ cpre,
                 const uint4* __restrict__ csuf, const uint4* __restrict__ ctot,
                 int32_t* __restrict__ lo, int32_t* __restrict__ hi) {
  const int cnt = *cross_count;
  const int lane = threadIdx.x & 31;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < cnt;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int4 c = cross[w];
    const int64_t ca = c.y / TC, ce = c.z / TC;
    uint4 acc = lane == 0 ? box_union(csuf[c.y], cpre[c.z]) : box_empty();
    for (int64_t k = ca + 1 + lane; k < ce; k += 32) acc = box_union(acc, ctot[k]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      uint4 u;
      u.x = __shfl_xor_sync(0xffffffffu, acc.x, o); u.y = __shfl_xor_sync(0xffffffffu, acc.y, o);
      u.z = __shfl_xor_sync(0xffffffffu, acc.z, o); u.w = __shfl_xor_sync(0xffffffffu, acc.w, o);
      acc = box_union(acc, u);
    }
    if (lane == 0) store_box(acc, bs, nx, ny, nz, c.x, lo, hi);
  }
}

// height() (lbvh.py:128-144) on demand: parents from the child arrays, then a per-leaf climb
// with arrival counters (the second arrival at a node knows both subtree heights).
__global__ void k_parents(const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                          const int* __restrict__ info, int32_t* __restrict__ parent,
                          int32_t* __restrict__ visit) {
  const int64_t n = info[0];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  parent[left[i]] = (int32_t)i;
  parent[right[i]] = (int32_t)i;
  visit[i] = 0;
}

__global__ void k_height_climb(const int32_t* __restrict__ left,
                               const int32_t* __restrict__ right,
                               const int32_t* __restrict__ parent, int32_t* __restrict__ visit,
                               int32_t* __restrict__ hgt, int* __restrict__ info) {
  const int64_t n = info[0];
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n < 2 || p >= n) return;
  int64_t node = parent[n - 1 + p];
  while (true) {
    __threadfence();
    if (atomicAdd(&visit[node], 1) == 0) return;
    __threadfence();
    const int32_t l = __ldcg(left + node), r = __ldcg(right + node);
    const int hl = (l >= n - 1) ? 1 : __ldcg(hgt + l);
    const int hr = (r >= n - 1) ? 1 : __ldcg(hgt + r);
    const int h = 1 + max(hl, hr);
    __stcg(hgt + node, h);
    if (node == 0) {
      info[1] = h;
      return;
    }
    node = __ldcg(parent + node);
  }
}

struct TreeWs {
  uint64_t* keys;
  int32_t* parent;
  int32_t* visit;
  int32_t* hgt;
  int2* range;
};

static TreeWs take_tree(Bump& b, int64_t cap) {
  TreeWs t;
  t.keys = b.take<uint64_t>(cap);
  t.parent = b.take<int32_t>(std::max<int64_t>(2 * cap - 1, 1));
  t.visit = b.take<int32_t>(std::max<int64_t>(cap, 1));
  t.hgt = b.take<int32_t>(std::max<int64_t>(cap, 1));
  t.range = b.take<int2>(std::max<int64_t>(cap, 1));
  return t;
}

static int tree_and_refit(const TreeWs& w, int64_t cap, int32_t* lo, int32_t* hi,
                          int32_t* left, int32_t* right, int32_t* leaf_brick, int* info,
                          cudaStream_t st) {
  VS_CUDA(cudaMemsetAsync(w.visit, 0, std::max<int64_t>(cap, 1) * sizeof(int32_t), st),
          "memset visit");
  const unsigned g = (unsigned)std::max<int64_t>(cdiv(cap, 256), 1);
  k_karras<<<g, 256, 0, st>>>(w.keys, info, cap, left, right, leaf_brick, w.parent, w.range);
  VS_TRY(check_launch("k_karras"));
  k_refit_chunked<<<(unsigned)std::max<int64_t>(cdiv(cap, RC), 1), RC, 0, st>>>(
      lo, hi, left, right, w.parent, w.range, w.visit, w.hgt, info);
  return check_launch("k_refit_chunked");
}

}  // namespace vs

using namespace vs;

extern "C" {

static size_t bitmap_ws(int P, int64_t cap, uint32_t** off, uint32_t** codes, uint4** cpre,
                        uint4** csuf, uint4** ctot, int4** cross, int** ccount, uint32_t** samp,
                        void* base) {
  const int64_t ntiles = (int64_t)P * P * P / 512;
  Bump b(base);
  uint32_t* o = b.take<uint32_t>(ntiles + 1);
  const bool big = ntiles > (int64_t)SCAN_T * SCAN_PER;
  if (big) b.take<char>(scan_temp_bytes(ntiles + 1));
  uint32_t* c = b.take<uint32_t>(std::max<int64_t>(cap, 1));
  uint4* pr = b.take<uint4>(std::max<int64_t>(cap, 1));
  uint4* sf = b.take<uint4>(std::max<int64_t>(cap, 1));
  uint4* tt = b.take<uint4>(cdiv(std::max<int64_t>(cap, 1), TC));
  int4* cr = b.take<int4>(std::max<int64_t>(cap, 1));
  int* cc = b.take<int>(1);
  uint32_t* sp = b.take<uint32_t>(NSAMP);
  if (off) {
    *off = o; *codes = c; *cpre = pr; *csuf = sf; *ctot = tt; *cross = cr; *ccount = cc;
    *samp = sp;
  }
  return b.off + 256;
}

size_t vs_lbvh_workspace(int P, int64_t cap) {
  return bitmap_ws(P, cap, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                   nullptr, nullptr);
}

int vs_lbvh_from_bitmap(const uint32_t* bitmap, const uint32_t* tile_counts, int P, int bs,
                        int nx, int ny, int nz, int64_t cap, int32_t* lo, int32_t* hi,
                        int32_t* left, int32_t* right, int32_t* leaf_brick,
                        int32_t* brick_coords, uint32_t* brick_grid, int* info, void* ws,
                        size_t ws_bytes, vs_stream_t stream) {
  if (!bitmap || !tile_counts || !lo || !hi || !left || !right || !leaf_brick ||
      !brick_coords || !info || bs < 1 || P < 8 || cap < 1)
    return fail_arg("vs_lbvh_from_bitmap");
  if (ws_bytes < vs_lbvh_workspace(P, cap)) return VS_EWORKSPACE;
  cudaStream_t st = S(stream);
  const int64_t ntiles = (int64_t)P * P * P / 512;
  uint32_t *off, *codes;
  uint4 *cpre, *csuf, *ctot;
  int4* cross;
  int* ccount;
  uint32_t* samp;
  bitmap_ws(P, cap, &off, &codes, &cpre, &csuf, &ctot, &cross, &ccount, &samp, ws);
  if (ntiles <= (int64_t)SCAN_T * SCAN_PER) {
    k_tile_scan<<<1, SCAN_T, 0, st>>>(tile_counts, ntiles, off);
    VS_TRY(check_launch("k_tile_scan"));
  } else {  // exclusive scan over ntiles+1 entries; the extra (zero) entry yields the total n
    size_t sb = scan_temp_bytes(ntiles + 1);
    void* tmp = reinterpret_cast<char*>(off) + (((ntiles + 1) * 4 + 255) & ~int64_t(255));
    VS_CUDA(cudaMemcpyAsync(off, tile_counts, ntiles * 4, cudaMemcpyDeviceToDevice, st), "copy");
    VS_CUDA(cudaMemsetAsync(off + ntiles, 0, 4, st), "memset");
    VS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, sb, off, off, (int)(ntiles + 1), st), "scan");
  }
  const int nby = (ny + bs - 1) / bs, nbz = (nz + bs - 1) / bs;
  if (brick_grid) {
    const int64_t nbx = (nx + bs - 1) / bs;
    VS_CUDA(cudaMemsetAsync(brick_grid, 0, ((nbx * nby * nbz + 31) / 32) * 4, st),
            "memset brick grid");
  }
  const int64_t pairs = cdiv(ntiles, 2);
  k_leaves_coop<<<(unsigned)cdiv(pairs, LV_WARPS), LV_WARPS * 32, 0, st>>>(
      bitmap, off, bs, nx, ny, nz, nby, nbz, ntiles, codes, lo, hi, left, right, leaf_brick,
      brick_coords, brick_grid, info, ccount, samp);
  VS_TRY(check_launch("k_leaves_coop"));
  const int nsm = sm_count();
  const int64_t grid = std::min<int64_t>(cdiv(cap, TC), (int64_t)nsm * 4);
  const int samp_bytes = NSAMP * 4;
  VS_CUDA(cudaFuncSetAttribute(k_tree_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               samp_bytes), "k_tree_chunk smem");
  k_tree_chunk<<<(unsigned)std::max<int64_t>(grid, 1), TC, samp_bytes, st>>>(
      codes, info, bs, nx, ny, nz, brick_coords, lo, hi, left, right, leaf_brick, cpre, csuf, ctot,
      cross, ccount, samp);
  VS_TRY(check_launch("k_tree_chunk"));
  k_tree_cross<<<(unsigned)nsm, 256, 0, st>>>(cross, ccount, bs, nx, ny, nz, cpre, csuf, ctot,
                                               lo, hi);
  return check_launch("k_tree_cross");
}

size_t vs_lbvh_height_workspace(int64_t cap) {
  Bump b(nullptr);
  b.take<int32_t>(std::max<int64_t>(2 * cap, 1));
  b.take<int32_t>(std::max<int64_t>(cap, 1));
  b.take<int32_t>(std::max<int64_t>(cap, 1));
  return b.off + 256;
}

int vs_lbvh_height(const int32_t* left, const int32_t* right, int* info, int64_t cap, void* ws,
                   size_t ws_bytes, vs_stream_t stream) {
  if (!left || !right || !info || cap < 1) return fail_arg("vs_lbvh_height");
  if (ws_bytes < vs_lbvh_height_workspace(cap)) return VS_EWORKSPACE;
  cudaStream_t st = S(stream);
  Bump b(ws);
  int32_t* parent = b.take<int32_t>(std::max<int64_t>(2 * cap, 1));
  int32_t* visit = b.take<int32_t>(std::max<int64_t>(cap, 1));
  int32_t* hgt = b.take<int32_t>(std::max<int64_t>(cap, 1));
  const unsigned g = (unsigned)cdiv(cap, 256);
  k_parents<<<g, 256, 0, st>>>(left, right, info, parent, visit);
  VS_TRY(check_launch("k_parents"));
  k_height_climb<<<g, 256, 0, st>>>(left, right, parent, visit, hgt, info);
  return check_launch("k_height_climb");
}

size_t vs_lbvh_bricks_workspace(int64_t n) {
  Bump b(nullptr);
  b.take<uint64_t>(std::max<int64_t>(n, 1));
  b.take<int32_t>(std::max<int64_t>(n, 1));
  b.take<int32_t>(std::max<int64_t>(n, 1));
  b.take<char>(sort_temp_bytes(std::max<int64_t>(n, 1)));
  take_tree(b, std::max<int64_t>(n, 1));
  return b.off + 256;
}

int vs_lbvh_from_bricks(const int32_t* coords, const uint32_t* codes, int64_t n, int bs, int nx,
                        int ny, int nz, int32_t* lo, int32_t* hi, int32_t* left, int32_t* right,
                        int32_t* leaf_brick, int32_t* brick_coords, int* info, void* ws,
                        size_t ws_bytes, vs_stream_t stream) {
  if (n < 0 || !info || bs < 1) return fail_arg("vs_lbvh_from_bricks");
  if (n > 0 && (!coords || !codes || !lo || !hi || !left || !right || !leaf_brick ||
                !brick_coords))
    return fail_arg("vs_lbvh_from_bricks: null output");
  if (ws_bytes < vs_lbvh_bricks_workspace(n)) return VS_EWORKSPACE;
  cudaStream_t st = S(stream);
  if (n == 0) {
    const int z[2] = {0, 0};
    VS_CUDA(cudaMemcpyAsync(info, z, sizeof z, cudaMemcpyHostToDevice, st), "info");
    return 0;
  }
  const int64_t cap = n;
  Bump b(ws);
  uint64_t* keys_in = b.take<uint64_t>(cap);
  int32_t* vals_in = b.take<int32_t>(cap);
  int32_t* order = b.take<int32_t>(cap);
  size_t sb = sort_temp_bytes(cap);
  void* tmp = b.take<char>(sb);
  TreeWs w = take_tree(b, cap);
  const unsigned g = (unsigned)cdiv(n, 256);
  k_make_keys<<<g, 256, 0, st>>>(codes, n, keys_in, vals_in);
  VS_TRY(check_launch("k_make_keys"));
  VS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sb, keys_in, w.keys, vals_in, order, (int)n, 0,
                                          64, st),
          "SortPairs");
  k_leaves_from_sorted<<<g, 256, 0, st>>>(coords, order, n, bs, nx, ny, nz, lo, hi, left, right,
                                          leaf_brick, brick_coords, info);
  VS_TRY(check_launch("k_leaves_from_sorted"));
  return tree_and_refit(w, cap, lo, hi, left, right, leaf_brick, info, st);
}

}  // extern "C"
