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

size_t vs_lbvh_workspace(int P, int64_t cap) {
  const int64_t ntiles = (int64_t)P * P * P / 512;
  Bump b(nullptr);
  b.take<uint32_t>(ntiles + 1);
  b.take<char>(scan_temp_bytes(ntiles + 1));
  take_tree(b, cap);
  return b.off + 256;
}

int vs_lbvh_from_bitmap(const uint32_t* bitmap, const uint32_t* tile_counts, int P, int bs,
                        int nx, int ny, int nz, int64_t cap, int32_t* lo, int32_t* hi,
                        int32_t* left, int32_t* right, int32_t* leaf_brick,
                        int32_t* brick_coords, int* info, void* ws, size_t ws_bytes,
                        vs_stream_t stream) {
  if (!bitmap || !tile_counts || !lo || !hi || !left || !right || !leaf_brick ||
      !brick_coords || !info || bs < 1 || P < 8 || cap < 1)
    return fail_arg("vs_lbvh_from_bitmap");
  if (ws_bytes < vs_lbvh_workspace(P, cap)) return VS_EWORKSPACE;
  cudaStream_t st = S(stream);
  const int64_t ntiles = (int64_t)P * P * P / 512;
  Bump b(ws);
  uint32_t* off = b.take<uint32_t>(ntiles + 1);
  size_t sb = scan_temp_bytes(ntiles + 1);
  void* tmp = b.take<char>(sb);
  TreeWs w = take_tree(b, cap);
  // exclusive scan over ntiles+1 entries; the extra (zero) entry yields the total n.
  VS_CUDA(cudaMemcpyAsync(off, tile_counts, ntiles * 4, cudaMemcpyDeviceToDevice, st), "copy");
  VS_CUDA(cudaMemsetAsync(off + ntiles, 0, 4, st), "memset");
  VS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, sb, off, off, (int)(ntiles + 1), st), "scan");
  k_leaves_from_bitmap<<<(unsigned)cdiv(ntiles * 16, 256), 256, 0, st>>>(
      bitmap, off, bs, nx, ny, nz, ntiles, w.keys, lo, hi, left, right, leaf_brick, brick_coords,
      info);
  VS_TRY(check_launch("k_leaves_from_bitmap"));
  return tree_and_refit(w, cap, lo, hi, left, right, leaf_brick, info, st);
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
