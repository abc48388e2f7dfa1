// Level-synchronous k-d tree construction over the packed bit volume: build_kdtree
// (/root/reference/pkg/src/voxelskip/kdtree.py:387-498) with both plane searches.
//
// The reference recursion is depth-first; its decisions for a node depend only on the node's
// box (and the root volume), so every node of one tree level is decided in parallel here and
// the rows are renumbered to the reference's DFS preorder at the end (emit-before-recurse,
// left subtree first; kdtree.py:412-419, 479-484).
//
// Per level (one host synchronisation: the level's node count and work totals):
//   sweep builder (kdtree.py:148-230): for every node that may split, per-slab spans along
//     each axis -- k_spans_rows<X>/<Y>: warp per (node, slab, 64-row chunk), a row's z words
//     on one lane group, chunks merged with atomics, plus the (x,z) / (y,z) OR-projections;
//     k_spans_z: z-slab spans from the projections by per-bit ballots -- then k_decide, one
//     block per node: _axis_sweep's prefix/suffix tight boxes as block scans, the cost argmin
//     (first minimum; strict < across axes), the acceptance test cost < box volume, the
//     halting rule and the forced middle split; children are exact tight boxes.
//   binned builder (kdtree.py:268-381): per-cell tight boxes once (precompute_cell_boxes),
//     per level the cell-slab unions (k_cell_slabs; the coordinate filter that _cells_reduce's
//     Morton range accelerates), k_decide_binned (warp per node: _snapped_positions in IEEE
//     double, first strict minimum) and the exact leaf shrink from the bits (k_leaf_shrink).
//   k_emit_level: rows of the level, the next level's boxes (left then right) and their work
//     sizes (prep_node), scanned on the device (k_multi_scan).
// Finalisation: subtree sizes bottom-up, preorder numbers top-down, scatter rows.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace vs {

namespace cg = cooperative_groups;

constexpr int KD_FAR = 0x3fffffff;  // "no coordinate" sentinel for minima (kdtree.py:40 _FAR)

struct Box {
  int lo[3], hi[3];
};

__host__ __device__ inline int64_t box_vol(const Box& b) {
  return (int64_t)(b.hi[0] - b.lo[0]) * (b.hi[1] - b.lo[1]) * (b.hi[2] - b.lo[2]);
}

// Slab span: coordinates local to the node box, min = KD_FAR / max = -1 when empty.
struct Span {
  int mn1, mx1, mn2, mx2;
};

// Per-level offset arrays (exclusive prefixes over the level's nodes, entry n = total), all
// computed by prep_node when the level's boxes are emitted and scanned on the device.
enum {
  A_X = 0,   // x-slab spans (ext x) of nodes that search / force-split
  A_Y,       // y-slab spans
  A_Z,       // z-slab spans
  A_PXZ,     // (x, z-word) projection words: ex * wz
  A_PYZ,     // (y, z-word) projection words: ey * wz
  A_ZW,      // z-span work items: wz
  A_SCR,     // suffix-box scratch: max extent
  A_IX,      // x-pass work items: ex * chunks(ey)
  A_IY,      // y-pass work items: ey * chunks(ex)
  A_IZ,      // z-pass work items: wz * chunks of 32 projection rows
  A_C0,      // binned: cell slabs along x, y, z
  A_C1,
  A_C2,
  A_IC0,     // binned: cell-slab work items (slab x chunks of CELL_CHUNK cells), per axis
  A_IC1,
  A_IC2,
  KA
};

// Cells one cell-slab work item reduces (chunks of a big slab merge with atomics).
#ifndef VS_CELL_CHUNK
#define VS_CELL_CHUNK 1024
#endif
constexpr int CELL_CHUNK = VS_CELL_CHUNK;
#ifndef VS_SHRINK_WARP
#define VS_SHRINK_WARP 1  // binned leaves of bounded size: warp-per-leaf exact shrink
#endif
#ifndef VS_CS_CU
#define VS_CS_CU 1  // k_cell_slabs: cells in flight per lane
#endif

// Rows one x/y-pass work item covers (a node's slab is split into chunks of this many rows so
// the top levels of a big volume still spread over every SM; chunks merge with atomics).
constexpr int SPAN_CHUNK = 64;
// Slabs of at most one chunk are grouped SLAB_GROUP to a work item (per-item overhead dominates
// the deep levels' small nodes).
constexpr int SLAB_GROUP = 4;

// Work items of one row pass over a node: es slabs of er rows each.
__host__ __device__ __forceinline__ int64_t span_items(int es, int er) {
  const int nch = (er + SPAN_CHUNK - 1) / SPAN_CHUNK;
  return nch <= 1 ? (int64_t)((es + SLAB_GROUP - 1) / SLAB_GROUP) : (int64_t)es * nch;
}

struct KdLevel {
  int n;                      // nodes on this level
  const Box* box;             // node boxes
  const int64_t* off[KA];     // n+1 exclusive prefixes
};

__device__ __forceinline__ int wz_of(const Box& b) { return (b.hi[2] - b.lo[2] + 31) >> 5; }

// Local z word w of row `row` for a node spanning global z [z0, z1): bits z0+32w .. (masked).
__device__ __forceinline__ uint32_t local_word(const uint32_t* __restrict__ row, int z0, int z1,
                                               int w) {
  const int gz = z0 + 32 * w;
  const int gw = gz >> 5, sh = gz & 31;
  uint32_t v = __ldg(row + gw) >> sh;
  if (sh && gz + 32 - sh < z1) v |= __ldg(row + gw + 1) << (32 - sh);
  const int rem = z1 - gz;
  if (rem < 32) v &= (1u << rem) - 1u;
  return v;
}

__device__ __forceinline__ int find_node(const int64_t* __restrict__ off, int n, int64_t item) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// A level's work items in one contiguous range per block; each warp walks its items in
// increasing order (stride = warps per block) and finds an item's node by stepping forward
// from the previous item's node, so only the first item pays the binary search.
struct ItemWalker {
  const int64_t* off;
  int64_t it, end;
  int node, step;
  __device__ __forceinline__ ItemWalker(const int64_t* off_, int n, int64_t items) : off(off_) {
    step = (int)(blockDim.x >> 5);
    const int64_t chunk = (items + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = (int64_t)blockIdx.x * chunk;
    end = min(items, b0 + chunk);
    it = b0 + (threadIdx.x >> 5);
    node = it < end ? find_node(off, n, it) : 0;
  }
  __device__ __forceinline__ bool valid() const { return it < end; }
  __device__ __forceinline__ void advance() {
    it += step;
    if (it < end)
      while (off[node + 1] <= it) ++node;
  }
};

// Lanes per row: the smallest power of two >= the node's z word count.
__device__ __forceinline__ int group_width(int wz) {
  return wz <= 1 ? 1 : 1 << (32 - __clz(wz - 1));
}

// One slab's rows [r0, r1) of a span pass: OR of the (masked) z words, first / last nonzero
// row.  DIRECT: one stored word per lane; else two stored words shifted to a local word.
template <int U, bool DIRECT>
__device__ __forceinline__ void rows_or(const uint32_t* __restrict__ bits, int ny, int nzw, int ax,
                                        int slab, int x0, int y0, int r0, int r1, int G, int g,
                                        int gw, uint32_t gmask, int w0, int w1, int ssh,
                                        uint32_t wmask, uint32_t& acc, int& rmin, int& rmax) {
  for (int rb = r0; rb < r1; rb += G * U) {
    uint32_t lo[U], hi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = min(rb + u * G + g, r1 - 1);
      const int x = ax == 0 ? slab : x0 + r;
      const int y = ax == 0 ? y0 + r : slab;
      const uint32_t* row = bits + ((int64_t)x * ny + y) * nzw;
      lo[u] = __ldg(row + w0);
      if (!DIRECT) hi[u] = __ldg(row + w1);
    }
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = rb + u * G + g < r1;
      uint32_t w = lo[u];
      if (!DIRECT && ssh) w = (lo[u] >> ssh) | (hi[u] << (32 - ssh));
      v[u] = ok ? (w & wmask) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t m = __ballot_sync(0xffffffffu, v[u] != 0);
      if ((m >> (g * gw)) & gmask) {
        const int r = rb + u * G + g;
        rmin = min(rmin, r);
        rmax = max(rmax, r);
      }
      acc |= v[u];
    }
  }
}

// ---- slab spans along x (AX = 0, rows = y) or y (AX = 1, rows = x), and the matching
//      (slab, z-word) OR projection ------------------------------------------------------
// Warp per (node, slab, chunk of SPAN_CHUNK rows).  A row's z words are read by one group of
// lanes (coalesced: the row's bits are contiguous), 32 / width rows per warp step, four steps
// in flight.  Single-chunk slabs store their span; chunked slabs merge into the initialised
// span / projection with atomics.
template <int AX>
__global__ void __launch_bounds__(256) k_spans_rows(const uint32_t* __restrict__ bits, int ny,
                                                    int nzw, KdLevel L, int64_t items,
                                                    Span* __restrict__ span,
                                                    uint32_t* __restrict__ proj) {
  constexpr int AI = AX == 0 ? A_IX : A_IY, AS = AX == 0 ? A_X : A_Y,
                AP = AX == 0 ? A_PXZ : A_PYZ;
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  for (ItemWalker W(L.off[AI], L.n, items); W.valid(); W.advance()) {
    const int64_t it = W.it;
    const int i = W.node;
    const Box b = L.box[i];
    const int er = b.hi[1 - AX] - b.lo[1 - AX];
    const int nch = (er + SPAN_CHUNK - 1) / SPAN_CHUNK;
    const int es = b.hi[AX] - b.lo[AX];
    const int local = (int)(it - L.off[AI][i]);
    const int s0 = nch == 1 ? local * SLAB_GROUP : local / nch;
    const int c = nch == 1 ? 0 : local - s0 * nch;
    const int s1 = nch == 1 ? min(es, s0 + SLAB_GROUP) : s0 + 1;
    const int r0 = c * SPAN_CHUNK, r1 = min(er, r0 + SPAN_CHUNK);
    const int wz = wz_of(b);
    // z words as stored (global alignment): one load per word, first / last word masked;
    // the OR-projection is shifted to node-local words once per slab.  Nodes spanning more
    // than 32 stored words (nz > 1024) read two words per local word instead.
    const int gwa = b.lo[2] >> 5, sh = b.lo[2] & 31;
    const int nwg = ((b.hi[2] - 1) >> 5) - gwa + 1;
    const bool direct = nwg <= 32;
    const int gw = group_width(direct ? nwg : wz), G = 32 / gw;
    const int g = lane / gw, wl = lane & (gw - 1);
    const uint32_t gmask = gw == 32 ? 0xffffffffu : ((1u << gw) - 1u);
    // branch-free loads (clamped addresses, masked after) so all loads are in flight at once
    int w0, w1;
    uint32_t wmask;
    if (direct) {
      w0 = w1 = gwa + min(wl, nwg - 1);
      const int hb = b.hi[2] & 31;
      wmask = wl < nwg ? 0xffffffffu : 0u;
      if (wl == 0) wmask &= 0xffffffffu << sh;
      if (wl == nwg - 1 && hb) wmask &= (1u << hb) - 1u;
    } else {
      const int wc = min(wl, wz - 1);
      const int gz = b.lo[2] + 32 * wc, rem = b.hi[2] - gz;
      w0 = gz >> 5;
      w1 = min(w0 + 1, nzw - 1);
      wmask = wl < wz ? (rem < 32 ? (1u << rem) - 1u : 0xffffffffu) : 0u;
    }
    const int ssh = direct ? 0 : sh;
    for (int s = s0; s < s1; ++s) {
    const int slab = b.lo[AX] + s;
    uint32_t acc = 0;
    int rmin = KD_FAR, rmax = -1;
    if (direct)
      rows_or<U, true>(bits, ny, nzw, AX, slab, b.lo[0], b.lo[1], r0, r1, G, g, gw, gmask, w0, w1,
                       0, wmask, acc, rmin, rmax);
    else
      rows_or<U, false>(bits, ny, nzw, AX, slab, b.lo[0], b.lo[1], r0, r1, G, g, gw, gmask, w0,
                        w1, ssh, wmask, acc, rmin, rmax);
    for (int o = gw; o < 32; o <<= 1) {
      acc |= __shfl_xor_sync(0xffffffffu, acc, o);
      rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
      rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    }
    if (direct) {  // stored words -> node-local words
      const uint32_t nxt = __shfl_down_sync(0xffffffffu, acc, 1);
      if (sh) acc = (acc >> sh) | (wl + 1 < nwg ? nxt << (32 - sh) : 0u);
      if (wl >= wz) acc = 0u;
    }
    const uint32_t mz = __ballot_sync(0xffffffffu, acc != 0) & gmask;
    const int wf = mz ? __ffs(mz) - 1 : 0, wlst = mz ? 31 - __clz(mz) : 0;
    const uint32_t af = __shfl_sync(0xffffffffu, acc, wf), al = __shfl_sync(0xffffffffu, acc, wlst);
    Span sp{rmin, rmax, KD_FAR, -1};
    if (mz) {
      sp.mn2 = 32 * wf + __ffs(af) - 1;
      sp.mx2 = 32 * wlst + 31 - __clz(al);
    }
    Span* dst = span + L.off[AS][i] + s;
    uint32_t* pdst = proj + L.off[AP][i] + (int64_t)s * wz;
    if (nch == 1) {
      if (lane == 0) *dst = sp;
      if (lane < wz) pdst[lane] = acc;
    } else if (rmax >= 0) {
      if (lane == 0) {
        atomicMin(&dst->mn1, sp.mn1);
        atomicMax(&dst->mx1, sp.mx1);
        atomicMin(&dst->mn2, sp.mn2);
        atomicMax(&dst->mx2, sp.mx2);
      }
      if (lane < wz && acc) atomicOr(pdst + lane, acc);
    }
    }  // slabs of the item
  }
}

// Empty spans / projections for the chunked merge.
__global__ void k_span_init(Span* __restrict__ sx, int64_t nx_, Span* __restrict__ sy, int64_t ny_,
                            Span* __restrict__ sz, int64_t nz_, uint32_t* __restrict__ px,
                            int64_t npx, uint32_t* __restrict__ py, int64_t npy) {
  const Span e{KD_FAR, -1, KD_FAR, -1};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       j < max(max(max(nx_, ny_), nz_), max(npx, npy)); j += stride) {
    if (j < nx_) sx[j] = e;
    if (j < ny_) sy[j] = e;
    if (j < nz_) sz[j] = e;
    if (j < npx) px[j] = 0;
    if (j < npy) py[j] = 0;
  }
}

// ---- z-slab spans from the two projections: warp per (node, z word, 32 projection rows) ----
// Lane k owns local z bit 32w + k; one ballot per z bit present in the chunk gives the bit's
// first / last row.  Single-chunk nodes store, chunked nodes merge with atomics.
__device__ __forceinline__ void proj_chunk(const uint32_t* __restrict__ p, int wz, int e,
                                           int base, int lane, int& mn, int& mx) {
  mn = KD_FAR;
  mx = -1;
  const int r = base + lane;
  const uint32_t v = r < e ? p[(int64_t)r * wz] : 0u;
  uint32_t cor = __reduce_or_sync(0xffffffffu, v);
  while (cor) {
    const int k = __ffs(cor) - 1;
    cor &= cor - 1;
    const uint32_t bal = __ballot_sync(0xffffffffu, (v >> k) & 1u);
    if (lane == k) {
      mn = base + __ffs(bal) - 1;
      mx = base + 31 - __clz(bal);
    }
  }
}

__global__ void __launch_bounds__(256) k_spans_z(KdLevel L, int64_t items,
                                                 const uint32_t* __restrict__ pxz,
                                                 const uint32_t* __restrict__ pyz,
                                                 Span* __restrict__ span_z) {
  const int lane = threadIdx.x & 31;
  for (ItemWalker W(L.off[A_IZ], L.n, items); W.valid(); W.advance()) {
    const int64_t it = W.it;
    const int i = W.node;
    const Box b = L.box[i];
    const int wz = wz_of(b);
    const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
    const int nch = (max(ex, ey) + 31) >> 5;
    const int local = (int)(it - L.off[A_IZ][i]);
    const int w = local / nch, base = (local - w * nch) * 32;
    const int nzb = min(32, ez - 32 * w);
    Span sp;
    proj_chunk(pxz + L.off[A_PXZ][i] + w, wz, ex, base, lane, sp.mn1, sp.mx1);
    proj_chunk(pyz + L.off[A_PYZ][i] + w, wz, ey, base, lane, sp.mn2, sp.mx2);
    Span* dst = span_z + L.off[A_Z][i] + 32 * w + lane;
    if (nch == 1) {
      if (lane < nzb) *dst = sp;
    } else if (lane < nzb) {
      if (sp.mx1 >= 0) { atomicMin(&dst->mn1, sp.mn1); atomicMax(&dst->mx1, sp.mx1); }
      if (sp.mx2 >= 0) { atomicMin(&dst->mn2, sp.mn2); atomicMax(&dst->mx2, sp.mx2); }
    }
  }
}

// ---- per-node decision ------------------------------------------------------------------
struct KdParams {
  int deep;          // 0 shallow, 1 deep
  int mls;           // max_leaf_size, -1 none
  int binned;
  int bins, cs;
  int64_t root_vol;
  int subtrees;      // sweep builder: small nodes are finished by k_subtrees (1) or per level (0)
};

struct KdDecision {
  int axis;          // -1 leaf
  int plane;
  int nchild;        // bit0 left present, bit1 right present
  int dropped;       // binned leaf whose shrink is empty (no row)
  int sub;           // -1; SUB_DEFER: the node's subtree is built by k_subtrees
  Box left, right;   // global boxes
  Box leaf;          // leaf row box (binned: shrunk)
};

__device__ __forceinline__ bool halted(const KdParams& P, int64_t vol) {
  return P.deep ? vol <= 512 : vol * 10 <= P.root_vol;  // kdtree.py:421-424
}

// ---- subtree hand-off (sweep builder) -------------------------------------------------------
// A node whose box fits one CTA's shared memory (extents <= SUB_EXT, packed bits <= SUB_WORDS
// words) and that is not a leaf outright is built to completion -- its whole subtree, in the
// reference's DFS preorder -- by one CTA of k_subtrees instead of level by level: the deep
// levels of a tree are long chains of small nodes, where a level-synchronous pass costs a few
// launches and a host round trip per level.
constexpr int SUB_EXT = 128;
#ifndef VS_SUB_WORDS
#define VS_SUB_WORDS 2560  // hand-off bound (measured: 10240 / 5120 / 2560 / 1280; 2560 fastest)
#endif
constexpr int SUB_WORDS = VS_SUB_WORDS;
constexpr int SUB_DEFER = -2;

__device__ __forceinline__ bool defer_node(const KdParams& P, const Box& b) {
  if (P.binned || !P.subtrees) return false;
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
  if (ex > SUB_EXT || ey > SUB_EXT || ez > SUB_EXT) return false;
  if ((int64_t)ex * ey * ((ez + 31) >> 5) > SUB_WORDS) return false;
  const int mx = max(ex, max(ey, ez));
  return !halted(P, box_vol(b)) || (P.mls >= 0 && mx > P.mls);
}

// Row-order tight box (axis row, other1, other2) in local coordinates; empty if hi0 < 0.
struct RBox {
  int lo0, lo1, lo2, hi0, hi1, hi2;
};

__device__ __forceinline__ int64_t rvol(const RBox& r) {
  if (r.hi0 < 0) return 0;
  return (int64_t)(r.hi0 - r.lo0 + 1) * (r.hi1 - r.lo1 + 1) * (r.hi2 - r.lo2 + 1);
}

__device__ __forceinline__ RBox rb_empty() { return RBox{KD_FAR, KD_FAR, KD_FAR, -1, -1, -1}; }

__device__ __forceinline__ RBox rb_join(const RBox& a, const RBox& b) {
  return RBox{min(a.lo0, b.lo0), min(a.lo1, b.lo1), min(a.lo2, b.lo2),
              max(a.hi0, b.hi0), max(a.hi1, b.hi1), max(a.hi2, b.hi2)};
}

__device__ __forceinline__ RBox slab_box(const Span* __restrict__ sp, int s) {
  const Span v = sp[s];
  return v.mx1 >= 0 ? RBox{s, v.mn1, v.mn2, s, v.mx1, v.mx2} : rb_empty();
}

__device__ __forceinline__ RBox rb_shfl(const RBox& r, int src_lane) {
  return RBox{__shfl_sync(0xffffffffu, r.lo0, src_lane), __shfl_sync(0xffffffffu, r.lo1, src_lane),
              __shfl_sync(0xffffffffu, r.lo2, src_lane), __shfl_sync(0xffffffffu, r.hi0, src_lane),
              __shfl_sync(0xffffffffu, r.hi1, src_lane), __shfl_sync(0xffffffffu, r.hi2, src_lane)};
}

// Block of DT threads cooperates on one node (k_decide / k_best_plane).
constexpr int DT = 128;
constexpr int DW = DT / 32;

struct DecideSmem {
  RBox wbox[DW];
  int64_t wcost[DW];
  int wk[DW];
  RBox best_l, best_r;  // sweep_axis: tight boxes of [0, k) and [k, e) at the chosen cut
};

// Exclusive block scan (join) of one box per thread in thread order (rev = false) or in
// reverse thread order (rev = true).
__device__ RBox block_excl_scan(RBox x, bool rev, DecideSmem& sm) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  RBox inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    RBox u;
    u.lo0 = rev ? __shfl_down_sync(0xffffffffu, inc.lo0, o) : __shfl_up_sync(0xffffffffu, inc.lo0, o);
    u.lo1 = rev ? __shfl_down_sync(0xffffffffu, inc.lo1, o) : __shfl_up_sync(0xffffffffu, inc.lo1, o);
    u.lo2 = rev ? __shfl_down_sync(0xffffffffu, inc.lo2, o) : __shfl_up_sync(0xffffffffu, inc.lo2, o);
    u.hi0 = rev ? __shfl_down_sync(0xffffffffu, inc.hi0, o) : __shfl_up_sync(0xffffffffu, inc.hi0, o);
    u.hi1 = rev ? __shfl_down_sync(0xffffffffu, inc.hi1, o) : __shfl_up_sync(0xffffffffu, inc.hi1, o);
    u.hi2 = rev ? __shfl_down_sync(0xffffffffu, inc.hi2, o) : __shfl_up_sync(0xffffffffu, inc.hi2, o);
    if (rev ? lane + o < 32 : lane >= o) inc = rb_join(inc, u);
  }
  // exclusive within the warp: the neighbour's inclusive value
  RBox ex = rb_shfl(inc, rev ? min(lane + 1, 31) : max(lane - 1, 0));
  if (rev ? lane == 31 : lane == 0) ex = rb_empty();
  __syncthreads();
  if (rev ? lane == 0 : lane == 31) sm.wbox[warp] = inc;  // warp total
  __syncthreads();
  for (int w = 0; w < DW; ++w)
    if (rev ? w > warp : w < warp) ex = rb_join(ex, sm.wbox[w]);
  return ex;
}

__device__ RBox block_reduce(RBox r, DecideSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  r = RBox{__reduce_min_sync(0xffffffffu, r.lo0), __reduce_min_sync(0xffffffffu, r.lo1),
           __reduce_min_sync(0xffffffffu, r.lo2), __reduce_max_sync(0xffffffffu, r.hi0),
           __reduce_max_sync(0xffffffffu, r.hi1), __reduce_max_sync(0xffffffffu, r.hi2)};
  __syncthreads();
  if (lane == 0) sm.wbox[warp] = r;
  __syncthreads();
  RBox t = rb_empty();
  for (int w = 0; w < DW; ++w) t = rb_join(t, sm.wbox[w]);
  return t;
}

// Tight row-order box of slabs [s0, s1).
__device__ RBox range_box(const Span* __restrict__ sp, int s0, int s1, DecideSmem& sm) {
  RBox r = rb_empty();
  for (int s = s0 + (int)threadIdx.x; s < s1; s += DT) r = rb_join(r, slab_box(sp, s));
  return block_reduce(r, sm);
}

// Sweep one axis (kdtree.py:156-188): first-minimum cut k in 1..e-1 and its cost
// vol(tight [0,k)) + vol(tight [k,e)).  Thread t owns a contiguous run of slabs; suffix boxes
// go to `suf` (e entries), prefix boxes stay in registers.
__device__ void sweep_axis(const Span* __restrict__ sp, int e, RBox* __restrict__ suf,
                           DecideSmem& sm, int& best_k, int64_t& best_cost) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (e + DT - 1) / DT;
  const int s0 = min(e, t * per), s1 = min(e, s0 + per);
  RBox loc = rb_empty();
  for (int s = s0; s < s1; ++s) loc = rb_join(loc, slab_box(sp, s));
  RBox r = block_excl_scan(loc, true, sm);  // slabs after my run
  for (int s = s1 - 1; s >= s0; --s) {
    r = rb_join(r, slab_box(sp, s));
    suf[s] = r;
  }
  RBox pre = block_excl_scan(loc, false, sm);  // slabs before my run (syncs: suf visible)
  int64_t bc = INT64_MAX;
  int bk = 0;
  RBox bpre = rb_empty();
  for (int s = s0; s < s1; ++s) {
    pre = rb_join(pre, slab_box(sp, s));
    if (s + 1 < e) {
      const int64_t c = rvol(pre) + rvol(suf[s + 1]);
      if (c < bc) { bc = c; bk = s + 1; bpre = pre; }
    }
  }
  const int64_t my_c = bc;
  const int my_k = bk;
  for (int o = 16; o; o >>= 1) {
    const int64_t c2 = __shfl_xor_sync(0xffffffffu, bc, o);
    const int k2 = __shfl_xor_sync(0xffffffffu, bk, o);
    if (c2 < bc || (c2 == bc && k2 < bk)) { bc = c2; bk = k2; }
  }
  __syncthreads();
  if (lane == 0) { sm.wcost[warp] = bc; sm.wk[warp] = bk; }
  __syncthreads();
  bc = sm.wcost[0];
  bk = sm.wk[0];
  for (int w = 1; w < DW; ++w)
    if (sm.wcost[w] < bc || (sm.wcost[w] == bc && sm.wk[w] < bk)) { bc = sm.wcost[w]; bk = sm.wk[w]; }
  // the winner's boxes: the cut is the first minimum of the thread owning slab k-1
  if (my_c == bc && my_k == bk && bc != INT64_MAX) { sm.best_l = bpre; sm.best_r = suf[bk]; }
  __syncthreads();
  best_k = bk;
  best_cost = bc;
}

// Row order -> xyz (kdtree.py:38 _ROWS_TO_XYZ): axis a rows are (a, o1, o2).
__device__ __forceinline__ void others(int a, int& o1, int& o2) {
  o1 = a == 0 ? 1 : 0;
  o2 = a == 2 ? 1 : 2;
}

// (register-only: the axis selects components, no dynamically indexed arrays)
__device__ __forceinline__ Box to_global(const Box& node, int a, const RBox& r) {
  const int lx = a == 0 ? r.lo0 : r.lo1, hx = a == 0 ? r.hi0 : r.hi1;
  const int ly = a == 0 ? r.lo1 : (a == 1 ? r.lo0 : r.lo2);
  const int hy = a == 0 ? r.hi1 : (a == 1 ? r.hi0 : r.hi2);
  const int lz = a == 2 ? r.lo0 : r.lo2, hz = a == 2 ? r.hi0 : r.hi2;
  Box g;
  g.lo[0] = node.lo[0] + lx; g.hi[0] = node.lo[0] + hx + 1;
  g.lo[1] = node.lo[1] + ly; g.hi[1] = node.lo[1] + hy + 1;
  g.lo[2] = node.lo[2] + lz; g.hi[2] = node.lo[2] + hz + 1;
  return g;
}

// ---- binned search helpers ---------------------------------------------------------------
// Per cell-slab union of occupied cells' tight boxes (global voxel coords), lo = KD_FAR empty.
struct CBox {
  int lo[3], hi[3];
};

// _snapped_positions (kdtree.py:346-350) in IEEE double, no FMA.
__device__ int snapped_positions(int lo, int hi, int bins, int cs, int* out) {
  const double extent = (double)(hi - lo);
  const double step = __ddiv_rn(extent, (double)bins);
  int n = 0;
  for (int j = 1; j < bins; ++j) {
    const double raw = __dadd_rn((double)lo, __dmul_rn((double)j, step));
    const int64_t p = (int64_t)floor(__dadd_rn(__ddiv_rn(raw, (double)cs), 0.5)) * cs;
    if (lo < p && p < hi) {
      bool dup = false;
      for (int q = 0; q < n; ++q) dup |= out[q] == (int)p;
      if (!dup) out[n++] = (int)p;
    }
  }
  for (int a = 1; a < n; ++a)  // sort ascending
    for (int b = a; b > 0 && out[b - 1] > out[b]; --b) { int t = out[b]; out[b] = out[b - 1]; out[b - 1] = t; }
  return n;
}

// _cells_reduce of a region through the node's cell-slab unions along axis a: cells with
// coordinate c in [c0, c1] along a (other axes: the node's cell range), union clipped to
// the region.  Returns false for None.
__device__ bool cells_reduce_axis(const CBox* __restrict__ cslab, int node_c0, int c0, int c1,
                                  const Box& region, int lane, Box& out) {
  Box u;
  for (int k = 0; k < 3; ++k) { u.lo[k] = KD_FAR; u.hi[k] = -1; }
  for (int c = c0 + lane; c <= c1; c += 32) {
    const CBox v = cslab[c - node_c0];
    if (v.lo[0] != KD_FAR) {
      for (int k = 0; k < 3; ++k) { u.lo[k] = min(u.lo[k], v.lo[k]); u.hi[k] = max(u.hi[k], v.hi[k]); }
    }
  }
  for (int k = 0; k < 3; ++k) {  // warp reductions (redux.sync)
    u.lo[k] = __reduce_min_sync(0xffffffffu, u.lo[k]);
    u.hi[k] = __reduce_max_sync(0xffffffffu, u.hi[k]);
  }
  if (u.lo[0] == KD_FAR) return false;
  for (int k = 0; k < 3; ++k) {
    out.lo[k] = max(u.lo[k], region.lo[k]);
    out.hi[k] = min(u.hi[k], region.hi[k]);
    if (out.lo[k] >= out.hi[k]) return false;
  }
  return true;
}

struct BinnedCtx {
  const CBox* cslab[3];      // per-level cell-slab unions, per axis
  const int64_t* coff[3];    // per-node offsets into cslab
  int nc[3];
  const CBox* cells;         // per-cell tight boxes, C order (small nodes reduce these directly)
};

// Nodes with at most this many cells skip the per-level cell-slab unions: their region
// unions are reduced straight from the cell boxes by the deciding warp.
constexpr int SMALL_CELLS = 64;

__device__ __forceinline__ void node_cell_range(const Box& b, int cs, const int* nc, int a,
                                                int& c0, int& c1) {
  c0 = max(b.lo[a] / cs, 0);
  c1 = min((b.hi[a] - 1) / cs, nc[a] - 1);
}

// _cells_reduce(region) for a region inside node box b (uses the axis-a slab unions).
__device__ __forceinline__ bool cells_reduce(const BinnedCtx& B, int i, const Box& node, int a,
                                             const Box& region, int cs, int lane, Box& out) {
  int n0, n1;
  node_cell_range(node, cs, B.nc, a, n0, n1);
  // region's cell range along a (kdtree.py:329-331), clamped like the reference
  const int c0 = max(region.lo[a] / cs, 0);
  const int c1 = min((region.hi[a] - 1) / cs, B.nc[a] - 1);
  for (int k = 0; k < 3; ++k) {
    int r0 = max(region.lo[k] / cs, 0), r1 = min((region.hi[k] - 1) / cs, B.nc[k] - 1);
    if (r0 > r1) return false;
  }
  // the node's cell range per axis (scalars: no dynamically indexed local arrays)
  int x0, x1, y0, y1, z0, z1;
  node_cell_range(node, cs, B.nc, 0, x0, x1);
  node_cell_range(node, cs, B.nc, 1, y0, y1);
  node_cell_range(node, cs, B.nc, 2, z0, z1);
  if ((x1 - x0 + 1) * (y1 - y0 + 1) * (z1 - z0 + 1) <= SMALL_CELLS) {
    // direct: the node's cells with coordinate along a in [c0, c1] (other axes: the node's
    // cell range, which is the region's), unioned, clipped to the region
    const int s0 = max(c0, n0), s1 = min(c1, n1);
    if (a == 0) { x0 = s0; x1 = s1; } else if (a == 1) { y0 = s0; y1 = s1; } else { z0 = s0; z1 = s1; }
    int ulo0 = KD_FAR, ulo1 = KD_FAR, ulo2 = KD_FAR, uhi0 = -1, uhi1 = -1, uhi2 = -1;
    const int e1 = y1 - y0 + 1, e2 = z1 - z0 + 1;
    const int cnt = s1 < s0 ? 0 : (x1 - x0 + 1) * e1 * e2;
    for (int q = lane; q < cnt; q += 32) {
      const int cx = x0 + q / (e1 * e2), cy = y0 + (q / e2) % e1, cz = z0 + q % e2;
      const CBox v = B.cells[((int64_t)cx * B.nc[1] + cy) * B.nc[2] + cz];
      if (v.lo[0] != KD_FAR) {
        ulo0 = min(ulo0, v.lo[0]); ulo1 = min(ulo1, v.lo[1]); ulo2 = min(ulo2, v.lo[2]);
        uhi0 = max(uhi0, v.hi[0]); uhi1 = max(uhi1, v.hi[1]); uhi2 = max(uhi2, v.hi[2]);
      }
    }
    ulo0 = __reduce_min_sync(0xffffffffu, ulo0);  // warp reductions (redux.sync)
    ulo1 = __reduce_min_sync(0xffffffffu, ulo1);
    ulo2 = __reduce_min_sync(0xffffffffu, ulo2);
    uhi0 = __reduce_max_sync(0xffffffffu, uhi0);
    uhi1 = __reduce_max_sync(0xffffffffu, uhi1);
    uhi2 = __reduce_max_sync(0xffffffffu, uhi2);
    if (ulo0 == KD_FAR) return false;
    out.lo[0] = max(ulo0, region.lo[0]); out.hi[0] = min(uhi0, region.hi[0]);
    out.lo[1] = max(ulo1, region.lo[1]); out.hi[1] = min(uhi1, region.hi[1]);
    out.lo[2] = max(ulo2, region.lo[2]); out.hi[2] = min(uhi2, region.hi[2]);
    return out.lo[0] < out.hi[0] && out.lo[1] < out.hi[1] && out.lo[2] < out.hi[2];
  }
  return cells_reduce_axis(B.cslab[a] + B.coff[a][i], n0, max(c0, n0), min(c1, n1), region,
                           lane, out);
}

// A small node's cells (<= SMALL_CELLS = 64: two per lane) held in registers by the deciding
// warp, so every candidate region's _cells_reduce is a masked fold plus warp reductions (the
// same cell set as cells_reduce's direct path: the node's cells whose coordinate along the
// split axis lies in the region's cell range).
struct SmallCells {
  CBox v[2];
  int c[2][3];
  int n0[3], n1[3];  // the node's cell range per axis
  __device__ __forceinline__ void load(const BinnedCtx& B, const Box& b, int cs, int lane) {
    for (int k = 0; k < 3; ++k) node_cell_range(b, cs, B.nc, k, n0[k], n1[k]);
    const int e1 = n1[1] - n0[1] + 1, e2 = n1[2] - n0[2] + 1;
    const int cnt = (n1[0] - n0[0] + 1) * e1 * e2;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int q = lane + 32 * j;
      c[j][0] = n0[0] + q / (e1 * e2);
      c[j][1] = n0[1] + (q / e2) % e1;
      c[j][2] = n0[2] + q % e2;
      if (q < cnt) {
        v[j] = B.cells[((int64_t)c[j][0] * B.nc[1] + c[j][1]) * B.nc[2] + c[j][2]];
      } else {
        v[j].lo[0] = KD_FAR;
      }
    }
  }
  // _cells_reduce(region) for a region of the node cut along axis a
  __device__ __forceinline__ bool reduce(const BinnedCtx& B, int a, const Box& region, int cs,
                                         Box& out) const {
    for (int k = 0; k < 3; ++k) {
      const int r0 = max(region.lo[k] / cs, 0), r1 = min((region.hi[k] - 1) / cs, B.nc[k] - 1);
      if (r0 > r1) return false;
    }
    // axis-a operands by selects (no dynamically indexed local arrays)
    const int rlo = a == 0 ? region.lo[0] : (a == 1 ? region.lo[1] : region.lo[2]);
    const int rhi = a == 0 ? region.hi[0] : (a == 1 ? region.hi[1] : region.hi[2]);
    const int nca = a == 0 ? B.nc[0] : (a == 1 ? B.nc[1] : B.nc[2]);
    const int na0 = a == 0 ? n0[0] : (a == 1 ? n0[1] : n0[2]);
    const int na1 = a == 0 ? n1[0] : (a == 1 ? n1[1] : n1[2]);
    const int c0 = max(rlo / cs, 0), c1 = min((rhi - 1) / cs, nca - 1);
    const int s0 = max(c0, na0), s1 = min(c1, na1);
    int ulo0 = KD_FAR, ulo1 = KD_FAR, ulo2 = KD_FAR, uhi0 = -1, uhi1 = -1, uhi2 = -1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int ca = a == 0 ? c[j][0] : (a == 1 ? c[j][1] : c[j][2]);
      if (v[j].lo[0] != KD_FAR && ca >= s0 && ca <= s1) {
        ulo0 = min(ulo0, v[j].lo[0]); ulo1 = min(ulo1, v[j].lo[1]); ulo2 = min(ulo2, v[j].lo[2]);
        uhi0 = max(uhi0, v[j].hi[0]); uhi1 = max(uhi1, v[j].hi[1]); uhi2 = max(uhi2, v[j].hi[2]);
      }
    }
    ulo0 = __reduce_min_sync(0xffffffffu, ulo0);
    ulo1 = __reduce_min_sync(0xffffffffu, ulo1);
    ulo2 = __reduce_min_sync(0xffffffffu, ulo2);
    uhi0 = __reduce_max_sync(0xffffffffu, uhi0);
    uhi1 = __reduce_max_sync(0xffffffffu, uhi1);
    uhi2 = __reduce_max_sync(0xffffffffu, uhi2);
    if (ulo0 == KD_FAR) return false;
    out.lo[0] = max(ulo0, region.lo[0]); out.hi[0] = min(uhi0, region.hi[0]);
    out.lo[1] = max(ulo1, region.lo[1]); out.hi[1] = min(uhi1, region.hi[1]);
    out.lo[2] = max(ulo2, region.lo[2]); out.hi[2] = min(uhi2, region.hi[2]);
    return out.lo[0] < out.hi[0] && out.lo[1] < out.hi[1] && out.lo[2] < out.hi[2];
  }
};

// Slab spans of one axis staged in shared memory by k_decide (with the suffix boxes) when the
// node's extent along the axis is at most this.
constexpr int STAGE_SLABS = 1024;

// ---- the decision kernel: one block of DT threads per node ----------------------------------
template <bool STAGE>
__global__ void __launch_bounds__(DT) k_decide(KdLevel L, KdParams P,
                                               const Span* __restrict__ span_x,
                                               const Span* __restrict__ span_y,
                                               const Span* __restrict__ span_z,
                                               RBox* __restrict__ scratch, BinnedCtx B,
                                               KdDecision* __restrict__ out,
                                               int64_t* __restrict__ child_count) {
  __shared__ DecideSmem sm;
  __shared__ Span stage_sp[STAGE ? STAGE_SLABS : 1];
  __shared__ RBox stage_suf[STAGE ? STAGE_SLABS : 1];
  const int t = threadIdx.x;
  const int i = blockIdx.x;
  if (i >= L.n) return;
  const Box b = L.box[i];
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
  const int64_t vol = box_vol(b);
  KdDecision d;
  d.axis = -1; d.plane = -1; d.nchild = 0; d.dropped = 0; d.sub = -1; d.leaf = b;
  if (defer_node(P, b)) {  // built by k_subtrees
    if (t == 0) {
      d.sub = SUB_DEFER;
      out[i] = d;
      child_count[i] = 0;
    }
    return;
  }
  bool split = false;
  const Span* spx = span_x + L.off[A_X][i];
  const Span* spy = span_y + L.off[A_Y][i];
  const Span* spz = span_z + L.off[A_Z][i];
  // axis-selected operands without dynamically indexed (local-memory) arrays
  auto axis_span = [&](int a) { return a == 0 ? spx : (a == 1 ? spy : spz); };
  auto axis_ext = [&](int a) { return a == 0 ? ex : (a == 1 ? ey : ez); };
  auto axis_lo = [&](int a) { return a == 0 ? b.lo[0] : (a == 1 ? b.lo[1] : b.lo[2]); };
  auto split_boxes = [&](int a, int k, const RBox& l, const RBox& r) {
    d.axis = a; d.plane = axis_lo(a) + k;
    if (l.hi0 >= 0) { d.left = to_global(b, a, l); d.nchild |= 1; }
    if (r.hi0 >= 0) { d.right = to_global(b, a, r); d.nchild |= 2; }
  };
  auto split_at = [&](int a, int k) {
    const Span* sp = axis_span(a);
    const RBox l = range_box(sp, 0, k, sm);
    const RBox r = range_box(sp, k, axis_ext(a), sm);
    split_boxes(a, k, l, r);
  };
  if (!halted(P, vol)) {
    // _sweep_search + acceptance (kdtree.py:191-221, 431-439)
    RBox* suf = scratch + L.off[A_SCR][i];
    int ba = -1, bk = 0;
    int64_t bc = 0;
    RBox bl = rb_empty(), br = rb_empty();
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int e = a == 0 ? ex : (a == 1 ? ey : ez);
      if (e < 2) continue;
      int k;
      int64_t c;
      const Span* sp = a == 0 ? spx : (a == 1 ? spy : spz);
      if (STAGE && e <= STAGE_SLABS) {
        // stage the axis' spans (coalesced, all loads in flight) and keep the suffix boxes
        // on chip
        __syncthreads();
        Span v[STAGE_SLABS / DT];
#pragma unroll
        for (int j = 0; j < STAGE_SLABS / DT; ++j)
          if (t + j * DT < e) v[j] = sp[t + j * DT];
#pragma unroll
        for (int j = 0; j < STAGE_SLABS / DT; ++j)
          if (t + j * DT < e) stage_sp[t + j * DT] = v[j];
        __syncthreads();
        sweep_axis(stage_sp, e, stage_suf, sm, k, c);
      } else {
        sweep_axis(sp, e, suf, sm, k, c);
      }
      if (ba >= 0 && c >= bc) continue;
      ba = a; bk = k; bc = c; bl = sm.best_l; br = sm.best_r;
    }
    if (ba >= 0 && bc < vol) {
      split_boxes(ba, bk, bl, br);
      split = true;
    }
  }
  if (!split && P.mls >= 0) {
    // forced_split (kdtree.py:441-467): middle of the longest axis, exact children
    int a = 0, e = ex;
    if (ey > e) { a = 1; e = ey; }
    if (ez > e) { a = 2; e = ez; }
    if (e > P.mls) {
      split_at(a, e / 2);
      split = true;
    }
  }
  if (t == 0) {
    out[i] = d;
    child_count[i] = __popc(d.nchild);
  }
}

// ---- binned decisions: one warp per node (kdtree.py:353-368, 441-467) ----------------------
// CS = 8: the default 8^3 cells as a compile-time constant (the cell-coordinate divisions
// become shifts) and, for bins <= 8, the candidate cuts generated in registers in ascending
// order (the snapped raster is monotone in j, so the reference's sort is the identity and its
// de-duplication is "differs from the previous accepted cut"); divisions by powers of two in
// _snapped_positions are exact multiplications.  CS = 0: any cell size / bin count.
__device__ __forceinline__ double div_exact(double x, int d) {
  return (d & (d - 1)) == 0 ? __dmul_rn(x, 1.0 / (double)d) : __ddiv_rn(x, (double)d);
}

// WPN = 1: four nodes per 128-thread CTA (wide levels).  WPN > 1: one node per CTA of WPN
// warps (narrow levels: a few big nodes), the candidates dealt round-robin over the warps and
// the winner taken as (least cost, then first candidate) -- the reference's first strict
// minimum of the sequential scan.
template <int WPN>
struct BinnedBest {
  long long cost[WPN];
  int idx[WPN], axis[WPN], plane[WPN], has[WPN];
  Box lb[WPN], rb[WPN];
};
template <int CS, int WPN>
__global__ void __launch_bounds__(WPN == 1 ? 128 : 32 * WPN)
    k_decide_binned(KdLevel L, KdParams P, BinnedCtx B, KdDecision* __restrict__ out,
                    int64_t* __restrict__ child_count) {
  __shared__ BinnedBest<WPN> sbest;
  const int lane = threadIdx.x & 31;
  const int wid = WPN == 1 ? 0 : (int)(threadIdx.x >> 5);
  const int i = WPN == 1 ? (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5))
                         : (int)blockIdx.x;
  if (i >= L.n) return;
  const Box b = L.box[i];
  const int ext[3] = {b.hi[0] - b.lo[0], b.hi[1] - b.lo[1], b.hi[2] - b.lo[2]};
  const int64_t vol = box_vol(b);
  KdDecision d;
  d.axis = -1; d.plane = -1; d.nchild = 0; d.dropped = 0; d.sub = -1; d.leaf = b;
  bool split = false;
  const int cs = CS ? CS : P.cs;
  int nlo[3], nhi[3];
  for (int k = 0; k < 3; ++k) node_cell_range(b, cs, B.nc, k, nlo[k], nhi[k]);
  const bool small =
      (nhi[0] - nlo[0] + 1) * (nhi[1] - nlo[1] + 1) * (nhi[2] - nlo[2] + 1) <= SMALL_CELLS;
  SmallCells SC;
  if (small) SC.load(B, b, cs, lane);
  auto reduce = [&](int a, const Box& region, Box& o) {
    return small ? SC.reduce(B, a, region, cs, o)
                 : cells_reduce(B, i, b, a, region, cs, lane, o);
  };
  if (!halted(P, vol)) {
    // first strict minimum over (axis, position)
    int ba = -1, bp = 0, bi = 0, ncand = 0;
    int64_t bc = 0;
    Box bl, br;
    bool hl = false, hr = false;
    auto candidate = [&](int a, int p) {
      const int ci = ncand++;
      if (WPN > 1 && ci % WPN != wid) return;
      Box lreg = b, rreg = b, lb, rb;
      if (a == 0) { lreg.hi[0] = p; rreg.lo[0] = p; }
      else if (a == 1) { lreg.hi[1] = p; rreg.lo[1] = p; }
      else { lreg.hi[2] = p; rreg.lo[2] = p; }
      const bool l = reduce(a, lreg, lb);
      const bool r = reduce(a, rreg, rb);
      const int64_t c = (l ? box_vol(lb) : 0) + (r ? box_vol(rb) : 0);
      if (ba < 0 || c < bc) { ba = a; bp = p; bc = c; bi = ci; bl = lb; br = rb; hl = l; hr = r; }
    };
    if (CS && P.bins <= 8) {
      for (int a = 0; a < 3; ++a) {
        const int lo = a == 0 ? b.lo[0] : (a == 1 ? b.lo[1] : b.lo[2]);
        const int hi = a == 0 ? b.hi[0] : (a == 1 ? b.hi[1] : b.hi[2]);
        const double step = div_exact((double)(hi - lo), P.bins);
        int last = INT_MIN;
#pragma unroll 1
        for (int j = 1; j < P.bins; ++j) {
          const double raw = __dadd_rn((double)lo, __dmul_rn((double)j, step));
          const int64_t p = (int64_t)floor(__dadd_rn(div_exact(raw, cs), 0.5)) * cs;
          if (lo < p && p < hi && (int)p != last) {
            last = (int)p;
            candidate(a, (int)p);
          }
        }
      }
    } else {
      for (int a = 0; a < 3; ++a) {
        int pos[64];
        const int np = snapped_positions(b.lo[a], b.hi[a], P.bins, cs, pos);
        for (int q = 0; q < np; ++q) candidate(a, pos[q]);
      }
    }
    if (WPN > 1) {  // combine the warps' bests: least cost, then first candidate
      if (lane == 0) {
        sbest.cost[wid] = bc; sbest.idx[wid] = bi; sbest.axis[wid] = ba; sbest.plane[wid] = bp;
        sbest.has[wid] = (hl ? 1 : 0) | (hr ? 2 : 0);
        sbest.lb[wid] = bl; sbest.rb[wid] = br;
      }
      __syncthreads();
      int w = -1;
      for (int k = 0; k < WPN; ++k)
        if (sbest.axis[k] >= 0 &&
            (w < 0 || sbest.cost[k] < sbest.cost[w] ||
             (sbest.cost[k] == sbest.cost[w] && sbest.idx[k] < sbest.idx[w])))
          w = k;
      if (wid != 0) return;
      ba = -1;
      if (w >= 0) {
        ba = sbest.axis[w]; bp = sbest.plane[w]; bc = sbest.cost[w];
        hl = sbest.has[w] & 1; hr = (sbest.has[w] >> 1) & 1;
        bl = sbest.lb[w]; br = sbest.rb[w];
      }
    }
    if (ba >= 0 && bc < vol) {
      d.axis = ba; d.plane = bp;
      if (hl) { d.left = bl; d.nchild |= 1; }
      if (hr) { d.right = br; d.nchild |= 2; }
      split = true;
    }
  }
  if (WPN > 1 && wid != 0) return;
  if (!split && P.mls >= 0) {
    // forced_split snapped to the interior raster
    int a = 0;
    if (ext[1] > ext[a]) a = 1;
    if (ext[2] > ext[a]) a = 2;
    if (ext[a] > P.mls) {
      const int lo = b.lo[a], hi = b.hi[a];
      int pos = lo + ext[a] / 2;
      const int first = (lo / cs + 1) * cs, last = ((hi - 1) / cs) * cs;
      if (first <= last) {
        const int64_t snap =
            (int64_t)floor(__dadd_rn(div_exact((double)pos, cs), 0.5)) * cs;
        const int64_t q = snap < first ? (int64_t)first : snap;
        pos = (int)(q > last ? (int64_t)last : q);
      }
      Box lreg = b, rreg = b, lb, rb;
      lreg.hi[a] = pos;
      rreg.lo[a] = pos;
      const bool l = reduce(a, lreg, lb);
      const bool r = reduce(a, rreg, rb);
      d.axis = a; d.plane = pos;
      if (l) { d.left = lb; d.nchild |= 1; }
      if (r) { d.right = rb; d.nchild |= 2; }
    }
  }
  if (lane == 0) {
    out[i] = d;
    child_count[i] = __popc(d.nchild);
  }
}

// ---- cell boxes (precompute_cell_boxes, kdtree.py:285-320) ---------------------------------
__global__ void k_cell_boxes(const uint32_t* __restrict__ bits, int nx, int ny, int nz, int cs,
                             int ncx, int ncy, int ncz, CBox* __restrict__ cells) {
  const int64_t n = (int64_t)ncx * ncy * ncz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cz = (int)(i % ncz), cy = (int)((i / ncz) % ncy), cx = (int)(i / ((int64_t)ncz * ncy));
  const int nzw = (int)nzw_of(nz);
  const int x0 = cx * cs, x1 = min(nx, x0 + cs), y0 = cy * cs, y1 = min(ny, y0 + cs);
  const int z0 = cz * cs, z1 = min(nz, z0 + cs);
  CBox c;
  for (int k = 0; k < 3; ++k) { c.lo[k] = KD_FAR; c.hi[k] = -1; }
  for (int x = x0; x < x1; ++x)
    for (int y = y0; y < y1; ++y) {
      const uint32_t* row = bits + ((int64_t)x * ny + y) * nzw;
      for (int w = z0 >> 5; w <= (z1 - 1) >> 5; ++w) {
        uint32_t v = __ldg(row + w);
        const int wb = w * 32;
        if (wb < z0) v &= 0xffffffffu << (z0 - wb);
        if (z1 - wb < 32) v &= (1u << (z1 - wb)) - 1u;
        if (!v) continue;
        c.lo[0] = min(c.lo[0], x); c.hi[0] = max(c.hi[0], x + 1);
        c.lo[1] = min(c.lo[1], y); c.hi[1] = max(c.hi[1], y + 1);
        c.lo[2] = min(c.lo[2], wb + __ffs(v) - 1);
        c.hi[2] = max(c.hi[2], wb + 32 - __clz(v));
      }
    }
  if (c.hi[0] < 0) c.lo[0] = KD_FAR;
  cells[i] = c;
}

// 8^3 cells (the binned builder's default): warp per (cell column cx, cy; 32 z words), lane
// = one z word = four cells.  The 64 rows of the column stream through coalesced loads; the
// cells' x / y / z occupancy comes out of per-byte "any" masks (SWAR), no per-voxel work.
__device__ __forceinline__ uint32_t bytes_any(uint32_t v) {  // 0x80 per nonzero byte
  return (((v & 0x7f7f7f7fu) + 0x7f7f7f7fu) | v) & 0x80808080u;
}
__global__ void __launch_bounds__(256) k_cell_boxes8(const uint32_t* __restrict__ bits, int nx,
                                                     int ny, int nz, int ncx, int ncy, int ncz,
                                                     CBox* __restrict__ cells) {
  const int nzw = (int)nzw_of(nz), nch = (nzw + 31) >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= (int64_t)ncx * ncy * nch) return;
  const int lane = threadIdx.x & 31;
  const int ch = (int)(warp % nch);
  const int cy = (int)((warp / nch) % ncy), cx = (int)(warp / ((int64_t)nch * ncy));
  const int w = 32 * ch + lane;
  if (w >= nzw) return;
  const uint32_t zm = nz - 32 * w >= 32 ? 0xffffffffu : (1u << (nz - 32 * w)) - 1u;
  const int x0 = 8 * cx, y0 = 8 * cy;
  const int lxn = min(8, nx - x0), lyn = min(8, ny - y0);
  uint32_t oy[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t xm = 0;
  for (int lx = 0; lx < lxn; ++lx) {
    const uint32_t* row = bits + ((int64_t)(x0 + lx) * ny + y0) * nzw + w;
    uint32_t v[8];
#pragma unroll
    for (int ly = 0; ly < 8; ++ly) v[ly] = ly < lyn ? __ldg(row + (int64_t)ly * nzw) & zm : 0u;
    uint32_t ox = 0;
#pragma unroll
    for (int ly = 0; ly < 8; ++ly) { ox |= v[ly]; oy[ly] |= v[ly]; }
    xm |= (bytes_any(ox) >> 7) << lx;
  }
  uint32_t ym = 0, zo = 0;
#pragma unroll
  for (int ly = 0; ly < 8; ++ly) { ym |= (bytes_any(oy[ly]) >> 7) << ly; zo |= oy[ly]; }
  CBox* out = cells + ((int64_t)cx * ncy + cy) * ncz;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int cz = 4 * w + k;
    if (cz >= ncz) break;
    const uint32_t zb = (zo >> (8 * k)) & 0xffu;
    CBox c;
    if (zb) {
      const uint32_t xb = (xm >> (8 * k)) & 0xffu, yb = (ym >> (8 * k)) & 0xffu;
      c.lo[0] = x0 + __ffs(xb) - 1; c.hi[0] = x0 + 32 - __clz(xb);
      c.lo[1] = y0 + __ffs(yb) - 1; c.hi[1] = y0 + 32 - __clz(yb);
      c.lo[2] = 8 * cz + __ffs(zb) - 1; c.hi[2] = 8 * cz + 32 - __clz(zb);
    } else {
      for (int j = 0; j < 3; ++j) { c.lo[j] = KD_FAR; c.hi[j] = -1; }
    }
    out[cz] = c;
  }
}

int launch_cell_boxes(const uint32_t* bits, int nx, int ny, int nz, int cs, int ncx, int ncy,
                      int ncz, CBox* cells, cudaStream_t st) {
  if (cs == 8) {
    const int64_t warps = (int64_t)ncx * ncy * ((nzw_of(nz) + 31) >> 5);
    k_cell_boxes8<<<(unsigned)cdiv(warps * 32, 256), 256, 0, st>>>(bits, nx, ny, nz, ncx, ncy,
                                                                    ncz, cells);
  } else {
    k_cell_boxes<<<(unsigned)cdiv((int64_t)ncx * ncy * ncz, 128), 128, 0, st>>>(
        bits, nx, ny, nz, cs, ncx, ncy, ncz, cells);
  }
  return check_launch("k_cell_boxes");
}

// Cell-slab unions along axis A: warp per (node, cell slab c in the node's cell range, chunk
// of CELL_CHUNK cells of the slab); chunked slabs merge into initialised unions with atomics.
__global__ void __launch_bounds__(256) k_cell_slabs(const CBox* __restrict__ cells, int ncx,
                                                    int ncy, int ncz, int cs, int A, KdLevel L,
                                                    int64_t items, CBox* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int nc[3] = {ncx, ncy, ncz};
  const int64_t* off = L.off[A_C0 + A];
  const int64_t* ioff = L.off[A_IC0 + A];
  for (ItemWalker W(ioff, L.n, items); W.valid(); W.advance()) {
    const int64_t it = W.it;
    const int i = W.node;
    const Box b = L.box[i];
    int c0[3], c1[3];
    for (int k = 0; k < 3; ++k) node_cell_range(b, cs, nc, k, c0[k], c1[k]);
    int o1, o2;
    others(A, o1, o2);
    const int n1 = c1[o1] - c0[o1] + 1, n2 = c1[o2] - c0[o2] + 1;
    const int nch = (n1 * n2 + CELL_CHUNK - 1) / CELL_CHUNK;
    const int local = (int)(it - ioff[i]);
    const int s = local / nch, ch = local - s * nch;
    const int c = c0[A] + s;
    const int q0 = ch * CELL_CHUNK, q1 = min(n1 * n2, q0 + CELL_CHUNK);
    CBox u;
    for (int k = 0; k < 3; ++k) { u.lo[k] = KD_FAR; u.hi[k] = -1; }
    // cell index = c * stride(A) + (c0[o1] + q / n2) * stride(o1) + (c0[o2] + q % n2) * stride(o2)
    const int64_t sxz = (int64_t)ncy * ncz;
    auto stride = [&](int k) { return k == 0 ? sxz : (k == 1 ? (int64_t)ncz : (int64_t)1); };
    const int b1 = o1 == 0 ? c0[0] : (o1 == 1 ? c0[1] : c0[2]);
    const int b2 = o2 == 0 ? c0[0] : (o2 == 1 ? c0[1] : c0[2]);
    const int64_t st1 = stride(o1), st2 = stride(o2);
    const int64_t cbase = (int64_t)c * stride(A) + b1 * st1 + b2 * st2;
    constexpr int CU = VS_CS_CU;  // cells in flight per lane
    for (int qb = q0 + lane; qb < q1; qb += 32 * CU) {
      CBox v[CU];
#pragma unroll
      for (int j = 0; j < CU; ++j) {
        const int q = qb + 32 * j;
        if (q < q1) {
          v[j] = cells[cbase + (int64_t)(q / n2) * st1 + (int64_t)(q % n2) * st2];
        } else {
          v[j].lo[0] = KD_FAR;
        }
      }
#pragma unroll
      for (int j = 0; j < CU; ++j)
        if (v[j].lo[0] != KD_FAR)
          for (int k = 0; k < 3; ++k) {
            u.lo[k] = min(u.lo[k], v[j].lo[k]);
            u.hi[k] = max(u.hi[k], v[j].hi[k]);
          }
    }
    for (int k = 0; k < 3; ++k) {  // warp reductions (redux.sync)
      u.lo[k] = __reduce_min_sync(0xffffffffu, u.lo[k]);
      u.hi[k] = __reduce_max_sync(0xffffffffu, u.hi[k]);
    }
    CBox* dst = out + off[i] + s;
    if (nch == 1) {
      if (lane == 0) *dst = u;
    } else if (lane < 3 && u.lo[0] != KD_FAR) {
      atomicMin(&dst->lo[lane], u.lo[lane]);
      atomicMax(&dst->hi[lane], u.hi[lane]);
    }
  }
}

// Packed cell boxes for cells of at most 16 voxels per axis: one 32-bit word per cell, the
// box as offsets from the cell's corner (4 bits each: lo x/y/z, then hi-1 x/y/z); empty =
// ~0.  Two copies: [x][y][z] (the x- and y-slab passes read runs along z) and [z][x][y] (the
// z-slab pass reads runs along y), so every cell-slab pass streams 4 contiguous bytes per
// cell instead of a strided 24-byte CBox.
#ifndef VS_CELL_PK
#define VS_CELL_PK 1  // 0: the cell-slab passes read the 24-byte CBoxes (A/B builds)
#endif
#ifndef VS_CPK_CU
#define VS_CPK_CU 4
#endif
constexpr uint32_t CPK_EMPTY = 0xffffffffu;
constexpr int CPK_MAX_CS = VS_CELL_PK ? 16 : 0;
__global__ void k_cell_pack(const CBox* __restrict__ cells, int ncx, int ncy, int ncz, int cs,
                            uint32_t* __restrict__ pxyz, uint32_t* __restrict__ pzxy) {
  const int64_t n = (int64_t)ncx * ncy * ncz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cz = (int)(i % ncz), cy = (int)((i / ncz) % ncy), cx = (int)(i / ((int64_t)ncz * ncy));
  const CBox c = cells[i];
  uint32_t v = CPK_EMPTY;
  if (c.lo[0] != KD_FAR) {
    const int b[3] = {cx * cs, cy * cs, cz * cs};
    v = 0;
    for (int k = 0; k < 3; ++k)
      v |= (uint32_t)(c.lo[k] - b[k]) << (4 * k) | (uint32_t)(c.hi[k] - 1 - b[k]) << (12 + 4 * k);
  }
  pxyz[i] = v;
  pzxy[((int64_t)cz * ncx + cx) * ncy + cy] = v;
}

// k_cell_slabs over the packed cells: the same items, the same unions (so the same
// decisions), 4 coalesced bytes per cell.  The slab's cross-section (o1, o2) is walked as
// rows of o2-contiguous cells; lane positions advance by a precomputed (rows, cols) step.
template <int A>
__device__ __forceinline__ void cell_slabs_pk(const uint32_t* __restrict__ pxyz,
                                              const uint32_t* __restrict__ pzxy, int ncx, int ncy,
                                              int ncz, int cs, const KdLevel& L, int64_t items,
                                              CBox* __restrict__ out) {
  constexpr int o1 = A == 0 ? 1 : 0, o2 = A == 2 ? 1 : 2;
  constexpr int CU = VS_CPK_CU;  // cells in flight per lane
  const int lane = threadIdx.x & 31;
  const int nc[3] = {ncx, ncy, ncz};
  const int64_t* off = L.off[A_C0 + A];
  const int64_t* ioff = L.off[A_IC0 + A];
  const uint32_t* __restrict__ pk = A == 2 ? pzxy : pxyz;
  for (ItemWalker W(ioff, L.n, items); W.valid(); W.advance()) {
    const int i = W.node;
    const Box b = L.box[i];
    int c0[3], c1[3];
    for (int k = 0; k < 3; ++k) node_cell_range(b, cs, nc, k, c0[k], c1[k]);
    const int n1 = c1[o1] - c0[o1] + 1, n2 = c1[o2] - c0[o2] + 1;
    const int nch = (n1 * n2 + CELL_CHUNK - 1) / CELL_CHUNK;
    const int local = (int)(W.it - ioff[i]);
    const int s = local / nch, ch = local - s * nch;
    const int c = c0[A] + s;
    const int q0 = ch * CELL_CHUNK, q1 = min(n1 * n2, q0 + CELL_CHUNK);
    // row stride of the layout along o1 (o2 is contiguous) and the slab's base cell
    int64_t st1, base;
    if (A == 0) {
      st1 = ncz; base = ((int64_t)c * ncy + c0[1]) * ncz + c0[2];
    } else if (A == 1) {
      st1 = (int64_t)ncy * ncz; base = ((int64_t)c0[0] * ncy + c) * ncz + c0[2];
    } else {
      st1 = ncy; base = ((int64_t)c * ncx + c0[0]) * ncy + c0[1];
    }
    int r = (q0 + lane) / n2, col = (q0 + lane) - r * n2;  // lane's first cell
    const int dr = 32 / n2, dc = 32 - dr * n2;              // one 32-cell step
    int ma_lo = 64, ma_hi = -1;                             // local offsets along A
    int m1_lo = KD_FAR, m1_hi = -1, m2_lo = KD_FAR, m2_hi = -1;
    for (int qb = q0 + lane; qb < q1; qb += 32 * CU) {
      uint32_t v[CU];
      int rr[CU], cc[CU];
#pragma unroll
      for (int j = 0; j < CU; ++j) {
        rr[j] = r; cc[j] = col;
        v[j] = qb + 32 * j < q1 ? __ldg(pk + base + (int64_t)r * st1 + col) : CPK_EMPTY;
        col += dc; r += dr;
        if (col >= n2) { col -= n2; ++r; }
      }
#pragma unroll
      for (int j = 0; j < CU; ++j)
        if (v[j] != CPK_EMPTY) {
          const int e1 = (c0[o1] + rr[j]) * cs, e2 = (c0[o2] + cc[j]) * cs;
          ma_lo = min(ma_lo, (int)(v[j] >> (4 * A)) & 15);
          ma_hi = max(ma_hi, (int)(v[j] >> (12 + 4 * A)) & 15);
          m1_lo = min(m1_lo, e1 + (int)((v[j] >> (4 * o1)) & 15));
          m1_hi = max(m1_hi, e1 + (int)((v[j] >> (12 + 4 * o1)) & 15));
          m2_lo = min(m2_lo, e2 + (int)((v[j] >> (4 * o2)) & 15));
          m2_hi = max(m2_hi, e2 + (int)((v[j] >> (12 + 4 * o2)) & 15));
        }
    }
    ma_lo = __reduce_min_sync(0xffffffffu, ma_lo);
    ma_hi = __reduce_max_sync(0xffffffffu, ma_hi);
    m1_lo = __reduce_min_sync(0xffffffffu, m1_lo);
    m1_hi = __reduce_max_sync(0xffffffffu, m1_hi);
    m2_lo = __reduce_min_sync(0xffffffffu, m2_lo);
    m2_hi = __reduce_max_sync(0xffffffffu, m2_hi);
    CBox u;
    if (ma_hi < 0) {
      for (int k = 0; k < 3; ++k) { u.lo[k] = KD_FAR; u.hi[k] = -1; }
    } else {
      u.lo[A] = c * cs + ma_lo; u.hi[A] = c * cs + ma_hi + 1;
      u.lo[o1] = m1_lo; u.hi[o1] = m1_hi + 1;
      u.lo[o2] = m2_lo; u.hi[o2] = m2_hi + 1;
    }
    CBox* dst = out + off[i] + s;
    if (nch == 1) {
      if (lane == 0) *dst = u;
    } else if (lane < 3 && ma_hi >= 0) {
      atomicMin(&dst->lo[lane], u.lo[lane]);
      atomicMax(&dst->hi[lane], u.hi[lane]);
    }
  }
}

// The three axes' passes in one launch (blockIdx.y = axis; they are independent).
__global__ void __launch_bounds__(256) k_cell_slabs_pk3(const uint32_t* __restrict__ pxyz,
                                                        const uint32_t* __restrict__ pzxy,
                                                        int ncx, int ncy, int ncz, int cs,
                                                        KdLevel L, int64_t i0, int64_t i1,
                                                        int64_t i2, CBox* o0, CBox* o1, CBox* o2) {
  if (blockIdx.y == 0)
    cell_slabs_pk<0>(pxyz, pzxy, ncx, ncy, ncz, cs, L, i0, o0);
  else if (blockIdx.y == 1)
    cell_slabs_pk<1>(pxyz, pzxy, ncx, ncy, ncz, cs, L, i1, o1);
  else
    cell_slabs_pk<2>(pxyz, pzxy, ncx, ncy, ncz, cs, L, i2, o2);
}

__global__ void k_cbox_init(CBox* __restrict__ c, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
    for (int k = 0; k < 3; ++k) { c[j].lo[k] = KD_FAR; c[j].hi[k] = -1; }
}

// ---- level bookkeeping ----------------------------------------------------------------------
struct NodeRec {   // per node, global BFS id
  Box box;
  int axis, plane, left, right, dropped, level;
  int sub;         // -1, SUB_DEFER (level loop), then the subtree id (k_collect_sub)
};

// Per-node work sizes of a level (written where the node's box is emitted).
struct PrepCtx {
  KdParams P;
  int nc[3];
  int64_t* arr[KA];   // per-node sizes, scanned in place afterwards
};

__device__ __forceinline__ void prep_node(const PrepCtx& C, const Box& b, int64_t i) {
  const KdParams& P = C.P;
  const int ext[3] = {b.hi[0] - b.lo[0], b.hi[1] - b.lo[1], b.hi[2] - b.lo[2]};
  int64_t v[KA];
  for (int k = 0; k < KA; ++k) v[k] = 0;
  if (!P.binned) {
    const int mx = max(ext[0], max(ext[1], ext[2]));
    const bool need = !halted(P, box_vol(b)) || (P.mls >= 0 && mx > P.mls);
    if (need && !defer_node(P, b)) {
      const int wz = (ext[2] + 31) >> 5;
      v[A_X] = ext[0];
      v[A_Y] = ext[1];
      v[A_Z] = ext[2];
      v[A_PXZ] = (int64_t)ext[0] * wz;
      v[A_PYZ] = (int64_t)ext[1] * wz;
      v[A_ZW] = wz;
      v[A_SCR] = mx;
      v[A_IX] = span_items(ext[0], ext[1]);
      v[A_IY] = span_items(ext[1], ext[0]);
      v[A_IZ] = (int64_t)wz * ((max(ext[0], ext[1]) + 31) >> 5);
    }
  } else {
    int n[3];
    for (int a = 0; a < 3; ++a) {
      int c0, c1;
      node_cell_range(b, P.cs, C.nc, a, c0, c1);
      n[a] = c1 - c0 + 1;
    }
    if (n[0] * n[1] * n[2] > SMALL_CELLS) {  // small nodes reduce their cells directly
      for (int a = 0; a < 3; ++a) {
        int o1, o2;
        others(a, o1, o2);
        v[A_C0 + a] = n[a];
        v[A_IC0 + a] = (int64_t)n[a] * ((n[o1] * n[o2] + CELL_CHUNK - 1) / CELL_CHUNK);
      }
    }
  }
  for (int k = 0; k < KA; ++k) C.arr[k][i] = v[k];
}

// Root level: one box from the device bbox (empty volume -> zero nodes).
__global__ void k_root_level(const int* __restrict__ bb, Box* __restrict__ box, PrepCtx C,
                             int64_t* __restrict__ hdr) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Box r;
  for (int k = 0; k < 3; ++k) { r.lo[k] = bb[k]; r.hi[k] = bb[3 + k]; }
  const bool any = bb[3] >= 0;
  hdr[0] = any ? 1 : 0;
  if (any) {
    box[0] = r;
    C.P.root_vol = box_vol(r);
    prep_node(C, r, 0);
  }
}

// Rows of this level's nodes + the next level's boxes (left child first) and work sizes.
__global__ void k_emit_level(const KdDecision* __restrict__ dec, const int64_t* __restrict__ coff,
                             int n, int64_t base, int64_t next_base, int level,
                             NodeRec* __restrict__ rec, Box* __restrict__ next_box, PrepCtx C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const KdDecision d = dec[i];
  NodeRec r;
  r.box = d.leaf;  // internal rows keep the node box; binned leaves the shrunk box
  r.axis = d.axis;
  r.plane = d.plane;
  r.left = r.right = -1;
  r.dropped = d.dropped;
  r.level = level;
  r.sub = d.sub;
  int64_t o = coff[i];
  if (d.nchild & 1) {
    next_box[o] = d.left;
    prep_node(C, d.left, o);
    r.left = (int)(next_base + o);
    ++o;
  }
  if (d.nchild & 2) {
    next_box[o] = d.right;
    prep_node(C, d.right, o);
    r.right = (int)(next_base + o);
  }
  rec[base + i] = r;
}

// Binned leaves: exact shrink_to_occupied(box) (kdtree.py:474) read straight from the bits;
// empty -> dropped (no row).  Block per leaf, blocks striding over the level's nodes (most are
// not leaves: a block per node would be mostly launch cost).
__global__ void __launch_bounds__(128) k_leaf_shrink(const uint32_t* __restrict__ bits, int ny,
                                                     int nzw, KdLevel L,
                                                     KdDecision* __restrict__ dec) {
  __shared__ int red[6];
  for (int i = blockIdx.x; i < L.n; i += gridDim.x) {
  if (dec[i].axis >= 0) continue;
  const Box b = L.box[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x < 6) red[threadIdx.x] = threadIdx.x < 3 ? KD_FAR : -1;
  __syncthreads();
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1];
  const int wz = wz_of(b), gw = group_width(wz), G = 32 / gw;
  const int g = lane / gw, wl = lane & (gw - 1);
  const uint32_t gmask = gw == 32 ? 0xffffffffu : ((1u << gw) - 1u);
  const int64_t rows = (int64_t)ex * ey;
  int lo[3] = {KD_FAR, KD_FAR, KD_FAR}, hi[3] = {-1, -1, -1};
  uint32_t acc = 0;
  for (int64_t rb = (int64_t)warp * G; rb < rows; rb += (int64_t)nw * G) {
    const int64_t q = rb + g;
    uint32_t v = 0;
    int x = 0, y = 0;
    if (q < rows && wl < wz) {
      x = (int)(q / ey);
      y = (int)(q - (int64_t)x * ey);
      v = local_word(bits + ((int64_t)(b.lo[0] + x) * ny + b.lo[1] + y) * nzw, b.lo[2], b.hi[2], wl);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, v != 0);
    if (wl == 0 && ((m >> (g * gw)) & gmask)) {
      lo[0] = min(lo[0], x); hi[0] = max(hi[0], x);
      lo[1] = min(lo[1], y); hi[1] = max(hi[1], y);
    }
    acc |= v;
  }
  // z extent from the per-lane OR words
  for (int o = gw; o < 32; o <<= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
  const uint32_t mz = __ballot_sync(0xffffffffu, acc != 0) & gmask;
  const int wf = mz ? __ffs(mz) - 1 : 0, wlst = mz ? 31 - __clz(mz) : 0;
  const uint32_t af = __shfl_sync(0xffffffffu, acc, wf), al = __shfl_sync(0xffffffffu, acc, wlst);
  if (mz) {
    lo[2] = 32 * wf + __ffs(af) - 1;
    hi[2] = 32 * wlst + 31 - __clz(al);
  }
  for (int k = 0; k < 3; ++k) {  // warp reductions (redux.sync)
    lo[k] = __reduce_min_sync(0xffffffffu, lo[k]);
    hi[k] = __reduce_max_sync(0xffffffffu, hi[k]);
  }
  if (lane == 0 && hi[0] >= 0)
    for (int k = 0; k < 3; ++k) { atomicMin(&red[k], lo[k]); atomicMax(&red[3 + k], hi[k]); }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (red[3] < 0) {
      dec[i].dropped = 1;
    } else {
      Box t;
      for (int k = 0; k < 3; ++k) { t.lo[k] = b.lo[k] + red[k]; t.hi[k] = b.lo[k] + red[3 + k] + 1; }
      dec[i].leaf = t;
    }
  }
  __syncthreads();  // red[] is reused by the block's next leaf
  }
}

// The same shrink with a warp per leaf (four leaves per 128-thread block, no block barriers)
// for leaves bounded by a small max-leaf-size (every leaf extent <= mls <= 64: at most 4096
// rows), four rows per lane group in flight.
__global__ void __launch_bounds__(128) k_leaf_shrink_warp(const uint32_t* __restrict__ bits,
                                                          int ny, int nzw, KdLevel L,
                                                          KdDecision* __restrict__ dec) {
  const int lane = threadIdx.x & 31;
  const int nwt = (int)((gridDim.x * blockDim.x) >> 5);
  for (int i = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < L.n; i += nwt) {
    if (dec[i].axis >= 0) continue;
    const Box b = L.box[i];
    const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1];
    const int wz = wz_of(b), gw = group_width(wz), G = 32 / gw;
    const int g = lane / gw, wl = lane & (gw - 1);
    const uint32_t gmask = gw == 32 ? 0xffffffffu : ((1u << gw) - 1u);
    const int rows = ex * ey;
    int lo0 = KD_FAR, lo1 = KD_FAR, hi0 = -1, hi1 = -1;
    uint32_t acc = 0;
    constexpr int U = 4;
    for (int rb = 0; rb < rows; rb += G * U) {
      uint32_t v[U];
      int xs[U], ys[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = rb + u * G + g;
        v[u] = 0;
        xs[u] = 0;
        ys[u] = 0;
        if (q < rows && wl < wz) {
          xs[u] = q / ey;
          ys[u] = q - xs[u] * ey;
          v[u] = local_word(bits + ((int64_t)(b.lo[0] + xs[u]) * ny + b.lo[1] + ys[u]) * nzw,
                            b.lo[2], b.hi[2], wl);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t m = __ballot_sync(0xffffffffu, v[u] != 0);
        if (wl == 0 && ((m >> (g * gw)) & gmask)) {
          lo0 = min(lo0, xs[u]); hi0 = max(hi0, xs[u]);
          lo1 = min(lo1, ys[u]); hi1 = max(hi1, ys[u]);
        }
        acc |= v[u];
      }
    }
    for (int o = gw; o < 32; o <<= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
    const uint32_t mz = __ballot_sync(0xffffffffu, acc != 0) & gmask;
    lo0 = __reduce_min_sync(0xffffffffu, lo0);
    lo1 = __reduce_min_sync(0xffffffffu, lo1);
    hi0 = __reduce_max_sync(0xffffffffu, hi0);
    hi1 = __reduce_max_sync(0xffffffffu, hi1);
    const int wf = mz ? __ffs(mz) - 1 : 0, wlst = mz ? 31 - __clz(mz) : 0;
    const uint32_t af = __shfl_sync(0xffffffffu, acc, wf), al = __shfl_sync(0xffffffffu, acc, wlst);
    if (lane == 0) {
      if (hi0 < 0) {
        dec[i].dropped = 1;
      } else {
        Box t;
        t.lo[0] = b.lo[0] + lo0; t.hi[0] = b.lo[0] + hi0 + 1;
        t.lo[1] = b.lo[1] + lo1; t.hi[1] = b.lo[1] + hi1 + 1;
        t.lo[2] = b.lo[2] + 32 * wf + __ffs(af) - 1;
        t.hi[2] = b.lo[2] + 32 * wlst + 31 - __clz(al) + 1;
        dec[i].leaf = t;
      }
    }
  }
}

// Exclusive scans of up to KA int64 arrays of n entries in place (entry n = total, also copied
// to totals[j]); n read from the device.  Block per array, 1024 threads, 4 items per thread.
struct ScanSet {
  int64_t* a[KA + 1];
  int64_t* totals[KA + 1];
  int k;
};

constexpr int SCAN_PER = 4, SCAN_TILE = 1024 * SCAN_PER;

// Exclusive scan of a[base, min(base + SCAN_TILE, n)) in place, offset by carry (1024 threads);
// returns carry + the tile's sum (every thread).
__device__ int64_t scan_tile(int64_t* __restrict__ a, int64_t base, int64_t n, int64_t carry,
                             int64_t* wsum, int64_t* total_s) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t v[SCAN_PER], s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    const int64_t j = base + (int64_t)t * SCAN_PER + k;
    v[k] = j < n ? a[j] : 0;
    s += v[k];
  }
  int64_t incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = wsum[lane], wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    wsum[lane] = wi - w;  // exclusive warp offsets
  }
  __syncthreads();
  int64_t run = carry + wsum[warp] + incl - s;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    const int64_t j = base + (int64_t)t * SCAN_PER + k;
    if (j < n) a[j] = run;
    run += v[k];
  }
  __syncthreads();
  if (t == 1023) *total_s = run;
  __syncthreads();
  return *total_s;
}

// One block per array: the whole array in SCAN_TILE steps (narrow levels).
__global__ void __launch_bounds__(1024) k_multi_scan(ScanSet S, const int64_t* __restrict__ n_ptr,
                                                    int64_t n_host) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t total_s;
  const int64_t n = n_ptr ? *n_ptr : n_host;
  int64_t* a = S.a[blockIdx.x];
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += SCAN_TILE) carry = scan_tile(a, base, n, carry, wsum, &total_s);
  if (threadIdx.x == 0) {
    a[n] = carry;
    if (S.totals[blockIdx.x]) *S.totals[blockIdx.x] = carry;
  }
}

// Wide levels: block (tile c, array j).  Pass 1: tile sums; pass 2: each tile's carry is the sum
// of the earlier tiles' sums, then the tile scan; the tile holding element n-1 writes the total.
__global__ void __launch_bounds__(256) k_scan_sums(ScanSet S, const int64_t* __restrict__ n_ptr,
                                                   int64_t n_host, int64_t* __restrict__ part,
                                                   int nch) {
  __shared__ int64_t ws[8];
  const int64_t n = n_ptr ? *n_ptr : n_host;
  const int64_t* a = S.a[blockIdx.y];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
  for (int64_t j = base + threadIdx.x; j < min(n, base + SCAN_TILE); j += 256) s += a[j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    part[(int64_t)blockIdx.y * nch + blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_apply(ScanSet S, const int64_t* __restrict__ n_ptr,
                                                     int64_t n_host,
                                                     const int64_t* __restrict__ part, int nch) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t total_s;
  const int64_t n = n_ptr ? *n_ptr : n_host;
  int64_t* a = S.a[blockIdx.y];
  const int c = blockIdx.x;
  const int64_t base = (int64_t)c * SCAN_TILE;
  if (base >= n && !(n == 0 && c == 0)) return;
  int64_t s = 0;  // carry: the earlier tiles' sums
  for (int q = threadIdx.x; q < c; q += 1024) s += part[(int64_t)blockIdx.y * nch + q];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
  __syncthreads();
  int64_t carry = 0;
  for (int w = 0; w < 32; ++w) carry += wsum[w];
  __syncthreads();
  const int64_t run = scan_tile(a, base, n, carry, wsum, &total_s);
  if (threadIdx.x == 0 && base + SCAN_TILE >= n) {  // the last tile (or the empty array)
    a[n] = run;
    if (S.totals[blockIdx.y]) *S.totals[blockIdx.y] = run;
  }
}

// Root box: tight box of every set bit (shrink_to_occupied of the full volume).  Warp per
// chunk of rows, lanes over a row's words (coalesced).
__global__ void __launch_bounds__(256) k_bits_bbox(const uint32_t* __restrict__ bits, int nx,
                                                   int ny, int nz, int* __restrict__ bb) {
  const int nzw = (int)nzw_of(nz);
  const int lane = threadIdx.x & 31;
  const int gw = group_width(nzw), G = 32 / gw;
  const int g = lane / gw, wl = lane & (gw - 1);
  const uint32_t gmask = gw == 32 ? 0xffffffffu : ((1u << gw) - 1u);
  const int64_t nrows = (int64_t)nx * ny;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lo[2] = {KD_FAR, KD_FAR}, hi[2] = {-1, -1};
  uint32_t acc = 0;
  const int wc = min(wl, nzw - 1);
  for (int64_t rb = wid * G; rb < nrows; rb += nwarps * G * 4) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // branch-free clamped loads: all four in flight
      const int64_t r = rb + (int64_t)u * nwarps * G + g;
      v[u] = __ldg(bits + min(r, nrows - 1) * nzw + wc);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t r = rb + (int64_t)u * nwarps * G + g;
      v[u] = (r < nrows && wl < nzw) ? v[u] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t r = rb + (int64_t)u * nwarps * G + g;
      const uint32_t m = __ballot_sync(0xffffffffu, v[u] != 0);
      if ((m >> (g * gw)) & gmask) {
        const int x = (int)(r / ny), y = (int)(r - (int64_t)x * ny);
        lo[0] = min(lo[0], x); hi[0] = max(hi[0], x);
        lo[1] = min(lo[1], y); hi[1] = max(hi[1], y);
      }
      acc |= v[u];
    }
  }
  for (int o = gw; o < 32; o <<= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
  const uint32_t mz = __ballot_sync(0xffffffffu, acc != 0) & gmask;
  const int wf = mz ? __ffs(mz) - 1 : 0, wlst = mz ? 31 - __clz(mz) : 0;
  const uint32_t af = __shfl_sync(0xffffffffu, acc, wf), al = __shfl_sync(0xffffffffu, acc, wlst);
  int zlo = KD_FAR, zhi = -1;
  if (mz) {
    zlo = 32 * wf + __ffs(af) - 1;
    zhi = 32 * wlst + 31 - __clz(al);
  }
  for (int k = 0; k < 2; ++k) {  // warp reductions (redux.sync)
    lo[k] = __reduce_min_sync(0xffffffffu, lo[k]);
    hi[k] = __reduce_max_sync(0xffffffffu, hi[k]);
  }
  if (lane == 0 && hi[0] >= 0) {
    atomicMin(bb + 0, lo[0]); atomicMax(bb + 3, hi[0] + 1);
    atomicMin(bb + 1, lo[1]); atomicMax(bb + 4, hi[1] + 1);
    atomicMin(bb + 2, zlo); atomicMax(bb + 5, zhi + 1);
  }
}

// Finalisation: subtree sizes (bottom-up per level), preorder (top-down per level), rows.
// Rows under record r: its own row plus its children's subtrees; a deferred node's subtree
// (k_subtrees) counts as built.
__device__ __forceinline__ int rec_size(const NodeRec& r, const int* __restrict__ size,
                                        const int* __restrict__ sub_count) {
  if (r.dropped) return 0;
  if (r.sub >= 0) return sub_count[r.sub];
  int s = 1;
  if (r.left >= 0) s += size[r.left];
  if (r.right >= 0) s += size[r.right];
  return s;
}

__global__ void k_sizes(const NodeRec* __restrict__ rec, int64_t b0, int64_t b1,
                        const int* __restrict__ sub_count, int* __restrict__ size) {
  const int64_t i = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b1) return;
  size[i] = rec_size(rec[i], size, sub_count);
}

__global__ void k_preorder(const NodeRec* __restrict__ rec, int64_t b0, int64_t b1,
                           const int* __restrict__ size, int* __restrict__ pre) {
  const int64_t i = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b1) return;
  const NodeRec r = rec[i];
  if (r.dropped) return;
  const int p = pre[i];
  int nxt = p + 1;
  if (r.left >= 0 && size[r.left] > 0) { pre[r.left] = nxt; nxt += size[r.left]; }
  if (r.right >= 0 && size[r.right] > 0) pre[r.right] = nxt;
}

// Both passes for every level in one block (levels are few-thousand-node sets on deep trees,
// so a block-wide barrier per level replaces two launches per level).
__global__ void __launch_bounds__(1024) k_order_levels(const NodeRec* __restrict__ rec,
                                                       const int64_t* __restrict__ level_base,
                                                       int nlevels,
                                                       const int* __restrict__ sub_count,
                                                       int* __restrict__ size,
                                                       int* __restrict__ pre) {
  for (int l = nlevels - 1; l >= 0; --l) {
    const int64_t b0 = level_base[l], b1 = level_base[l + 1];
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
      size[i] = rec_size(rec[i], size, sub_count);
    __syncthreads();
  }
  if (threadIdx.x == 0) pre[0] = 0;
  __syncthreads();
  for (int l = 0; l < nlevels; ++l) {
    const int64_t b0 = level_base[l], b1 = level_base[l + 1];
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const NodeRec r = rec[i];
      if (r.dropped) continue;
      const int p = pre[i];
      int nxt = p + 1;
      if (r.left >= 0 && size[r.left] > 0) { pre[r.left] = nxt; nxt += size[r.left]; }
      if (r.right >= 0 && size[r.right] > 0) pre[r.right] = nxt;
    }
    __syncthreads();
  }
}

// The same two passes for big trees over a co-resident grid (cooperative launch), one grid
// barrier per level instead of two launches per level (the binned trees: 85K-680K rows over
// 24-32 levels at 1024^3).
__global__ void __launch_bounds__(1024) k_order_levels_grid(const NodeRec* __restrict__ rec,
                                                            const int64_t* __restrict__ level_base,
                                                            int nlevels,
                                                            const int* __restrict__ sub_count,
                                                            int* __restrict__ size,
                                                            int* __restrict__ pre) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int l = nlevels - 1; l >= 0; --l) {
    const int64_t b0 = level_base[l], b1 = level_base[l + 1];
    for (int64_t i = b0 + tid; i < b1; i += nth) size[i] = rec_size(rec[i], size, sub_count);
    grid.sync();
  }
  if (tid == 0) pre[0] = 0;
  grid.sync();
  for (int l = 0; l < nlevels; ++l) {
    const int64_t b0 = level_base[l], b1 = level_base[l + 1];
    for (int64_t i = b0 + tid; i < b1; i += nth) {
      const NodeRec r = rec[i];
      if (r.dropped) continue;
      const int p = pre[i];
      int nxt = p + 1;
      if (r.left >= 0 && size[r.left] > 0) { pre[r.left] = nxt; nxt += size[r.left]; }
      if (r.right >= 0 && size[r.right] > 0) pre[r.right] = nxt;
    }
    grid.sync();
  }
}

__global__ void k_scatter_rows(const NodeRec* __restrict__ rec, int64_t total,
                               const int* __restrict__ size, const int* __restrict__ pre,
                               int32_t* __restrict__ lo, int32_t* __restrict__ hi,
                               int8_t* __restrict__ axis, int32_t* __restrict__ plane,
                               int32_t* __restrict__ left, int32_t* __restrict__ right,
                               int* __restrict__ height) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const NodeRec r = rec[i];
  if (r.dropped || r.sub >= 0) return;  // deferred nodes: k_scatter_sub
  const int p = pre[i];
  for (int k = 0; k < 3; ++k) { lo[3 * p + k] = r.box.lo[k]; hi[3 * p + k] = r.box.hi[k]; }
  axis[p] = (int8_t)r.axis;
  plane[p] = r.plane;
  left[p] = (r.left >= 0 && size[r.left] > 0) ? pre[r.left] : -1;
  right[p] = (r.right >= 0 && size[r.right] > 0) ? pre[r.right] : -1;
  atomicMax(height, r.level + 1);
}

// ---- subtrees: one CTA builds a deferred node's whole subtree from shared memory ----------
// The node's packed bits are staged once (R-local rows, z words from the box's first z); the
// CTA then runs the reference recursion itself (kdtree.py:479-484: emit, then left subtree,
// then right) with an explicit stack, so rows come out in local DFS preorder.  Per node:
//   1. spans: warp per group of x slabs (lanes over y) -- x-slab spans and (x, z-word)
//      projections by segment reductions, y-slab spans and (y, z-word) projections by shared
//      atomics; z-slab spans from the projections (thread per z);
//   2. warps 0..2 sweep axes x, y, z (first-minimum cut, prefix / suffix tight boxes by warp
//      scans); warp 3 the forced middle split's exact boxes;
//   3. thread 0 decides (strict < across axes, cost < volume, else forced, else leaf), writes
//      the row and pushes right then left child.
// Rows go to a global pool in 32-row chunks (chunk table in shared memory, copied out at the
// end); k_scatter_sub places them once the global preorder is known.
constexpr int SUB_T = 128;
constexpr int SUB_STACK = 3 * SUB_EXT + 8;
constexpr int SUB_CHUNK = 32;
constexpr int SUB_MAXCH = 1024;  // 32768 rows per subtree

struct SubRow {
  int lo[3], hi[3];
  int axis, plane, left, right;
};

struct SubEntry {
  short lo[3], hi[3];
  int parent;
  short depth, right;
};

struct SubAxis {
  long long cost;
  int k, valid;
  RBox l, r;
};

struct SubSmem {
  Span spx[SUB_EXT], spy[SUB_EXT], spz[SUB_EXT];
  uint32_t pxz[SUB_EXT * 4], pyz[SUB_EXT * 4];
  SubEntry stack[SUB_STACK];
  int chunk[SUB_MAXCH];
  SubAxis ax[3], forced;
  SubEntry cur;
  int sp, count, maxdepth, status, choff;
};

struct SubCtx {
  const NodeRec* rec;
  const int* list;
  SubRow* pool;
  long long pool_chunks;              // capacity in chunks
  unsigned long long* pool_used;      // chunks handed out
  int* count;                         // rows per subtree
  int* height;                        // local height per subtree
  int* choff;                         // chunk-table offset per subtree
  int* chunks;                        // chunk tables, concatenated
  unsigned long long* chunks_used;
  int* status;                        // bit 0: pool exhausted, bit 1: a subtree too large
  const int* order;                   // launch order of the subtrees (nullptr: by id)
};

__device__ __forceinline__ RBox rb_shfl_up(const RBox& r, int o) {
  return RBox{__shfl_up_sync(0xffffffffu, r.lo0, o), __shfl_up_sync(0xffffffffu, r.lo1, o),
              __shfl_up_sync(0xffffffffu, r.lo2, o), __shfl_up_sync(0xffffffffu, r.hi0, o),
              __shfl_up_sync(0xffffffffu, r.hi1, o), __shfl_up_sync(0xffffffffu, r.hi2, o)};
}
__device__ __forceinline__ RBox rb_shfl_down(const RBox& r, int o) {
  return RBox{__shfl_down_sync(0xffffffffu, r.lo0, o), __shfl_down_sync(0xffffffffu, r.lo1, o),
              __shfl_down_sync(0xffffffffu, r.lo2, o), __shfl_down_sync(0xffffffffu, r.hi0, o),
              __shfl_down_sync(0xffffffffu, r.hi1, o), __shfl_down_sync(0xffffffffu, r.hi2, o)};
}
__device__ __forceinline__ RBox rb_warp_reduce(RBox r) {
  return RBox{__reduce_min_sync(0xffffffffu, r.lo0), __reduce_min_sync(0xffffffffu, r.lo1),
              __reduce_min_sync(0xffffffffu, r.lo2), __reduce_max_sync(0xffffffffu, r.hi0),
              __reduce_max_sync(0xffffffffu, r.hi1), __reduce_max_sync(0xffffffffu, r.hi2)};
}

// Slab spans of node b (R-local box) from the staged words: spx / spy / spz in node-local
// coordinates, as k_spans_rows / k_spans_z produce them.
__device__ void sub_spans(SubSmem& sm, const uint32_t* __restrict__ words, int eyR, int wzR,
                          const Box& b) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
  const int w0 = b.lo[2] >> 5, w1 = (b.hi[2] - 1) >> 5, nwz = w1 - w0 + 1;
  uint32_t m[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t v = w < nwz ? 0xffffffffu : 0u;
    if (w == 0) v &= 0xffffffffu << (b.lo[2] & 31);
    if (w == nwz - 1 && (b.hi[2] & 31)) v &= (1u << (b.hi[2] & 31)) - 1u;
    m[w] = v;
  }
  for (int i = t; i < ey; i += SUB_T) sm.spy[i] = Span{KD_FAR, -1, KD_FAR, -1};
  for (int i = t; i < ey * nwz; i += SUB_T) sm.pyz[i] = 0u;
  __syncthreads();
  // x slabs: lane groups of gw lanes (pow2 >= ey, <= 32), G = 32 / gw slabs per warp step
  const int gw = ey >= 32 ? 32 : group_width(ey), G = 32 / gw;
  const int g = lane / gw, yl = lane & (gw - 1);
  for (int xb = warp * G; xb < ex; xb += (SUB_T / 32) * G) {
    const int x = xb + g;
    int ymn = KD_FAR, ymx = -1, zmn = KD_FAR, zmx = -1;
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    if (x < ex) {
      for (int y = yl; y < ey; y += gw) {
        const uint32_t* row = words + ((b.lo[0] + x) * eyR + b.lo[1] + y) * wzR + w0;
        uint32_t v[4];
        int zl = KD_FAR, zh = -1;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          v[w] = w < nwz ? row[w] & m[w] : 0u;
          o[w] |= v[w];
        }
#pragma unroll
        for (int w = 3; w >= 0; --w)
          if (v[w]) zl = 32 * (w0 + w) + __ffs(v[w]) - 1;
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (v[w]) zh = 32 * (w0 + w) + 31 - __clz(v[w]);
        if (zh >= 0) {
          zl -= b.lo[2];
          zh -= b.lo[2];
          ymn = min(ymn, y);
          ymx = max(ymx, y);
          zmn = min(zmn, zl);
          zmx = max(zmx, zh);
          Span* d = &sm.spy[y];
          atomicMin(&d->mn1, x);
          atomicMax(&d->mx1, x);
          atomicMin(&d->mn2, zl);
          atomicMax(&d->mx2, zh);
#pragma unroll
          for (int w = 0; w < 4; ++w)
            if (v[w]) atomicOr(&sm.pyz[y * nwz + w], v[w]);
        }
      }
    }
    for (int off = 1; off < gw; off <<= 1) {
      ymn = min(ymn, __shfl_xor_sync(0xffffffffu, ymn, off));
      ymx = max(ymx, __shfl_xor_sync(0xffffffffu, ymx, off));
      zmn = min(zmn, __shfl_xor_sync(0xffffffffu, zmn, off));
      zmx = max(zmx, __shfl_xor_sync(0xffffffffu, zmx, off));
#pragma unroll
      for (int w = 0; w < 4; ++w) o[w] |= __shfl_xor_sync(0xffffffffu, o[w], off);
    }
    if (yl == 0 && x < ex) {
      sm.spx[x] = Span{ymn, ymx, zmn, zmx};
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (w < nwz) sm.pxz[x * nwz + w] = o[w];
    }
  }
  __syncthreads();
  // z slabs from the projections: first / last x (y) whose projection holds the z bit
  for (int z = t; z < ez; z += SUB_T) {
    const int zr = b.lo[2] + z, wi = (zr >> 5) - w0, bit = zr & 31;
    Span sp{KD_FAR, -1, KD_FAR, -1};
    int x = 0;
    while (x < ex && !((sm.pxz[x * nwz + wi] >> bit) & 1u)) ++x;
    if (x < ex) {
      sp.mn1 = x;
      x = ex - 1;
      while (!((sm.pxz[x * nwz + wi] >> bit) & 1u)) --x;
      sp.mx1 = x;
      int y = 0;
      while (!((sm.pyz[y * nwz + wi] >> bit) & 1u)) ++y;
      sp.mn2 = y;
      y = ey - 1;
      while (!((sm.pyz[y * nwz + wi] >> bit) & 1u)) --y;
      sp.mx2 = y;
    }
    sm.spz[z] = sp;
  }
  __syncthreads();
}

// _axis_sweep + first-minimum cut for one axis (one warp; e <= SUB_EXT: four slabs per lane).
__device__ void sub_sweep_axis(const Span* __restrict__ sp, int e, SubAxis& out) {
  const int lane = threadIdx.x & 31;
  if (e < 2) {
    if (lane == 0) out.valid = 0;
    return;
  }
  const int per = (e + 31) >> 5;
  const int s0 = min(e, lane * per), s1 = min(e, s0 + per);
  RBox sb[4];
  RBox loc = rb_empty();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    sb[j] = s0 + j < s1 ? slab_box(sp, s0 + j) : rb_empty();
    loc = rb_join(loc, sb[j]);
  }
  // inclusive scans of the lane runs: prefix (up) and suffix (down)
  RBox pin = loc, sin = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const RBox u = rb_shfl_up(pin, o), d = rb_shfl_down(sin, o);
    if (lane >= o) pin = rb_join(pin, u);
    if (lane + o < 32) sin = rb_join(sin, d);
  }
  RBox before = rb_shfl_up(pin, 1), after = rb_shfl_down(sin, 1);
  if (lane == 0) before = rb_empty();
  if (lane == 31) after = rb_empty();
  RBox suf[5];
  suf[4] = after;
#pragma unroll
  for (int j = 3; j >= 0; --j) suf[j] = s0 + j < s1 ? rb_join(sb[j], suf[j + 1]) : suf[j + 1];
  long long bc = LLONG_MAX;
  int bk = 0, bj = -1;
  RBox pre = before;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (s0 + j < s1) {
      pre = rb_join(pre, sb[j]);
      if (s0 + j + 1 < e) {
        const long long c = rvol(pre) + rvol(suf[j + 1]);
        if (c < bc) { bc = c; bk = s0 + j + 1; bj = j; }
      }
    }
  }
  long long wc = bc;
  int wk = bk;
  for (int o = 16; o; o >>= 1) {
    const long long c2 = __shfl_xor_sync(0xffffffffu, wc, o);
    const int k2 = __shfl_xor_sync(0xffffffffu, wk, o);
    if (c2 < wc || (c2 == wc && k2 < wk)) { wc = c2; wk = k2; }
  }
  if (bj >= 0 && bc == wc && bk == wk) {  // the winner: prefix through k-1, suffix from k
    RBox l = before;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j <= bj) l = rb_join(l, sb[j]);
    RBox r = suf[4];
#pragma unroll
    for (int j = 3; j >= 0; --j)
      if (j > bj && s0 + j < s1) r = rb_join(r, sb[j]);
    out.cost = wc;
    out.k = wk;
    out.valid = 1;
    out.l = l;
    out.r = r;
  }
}

// forced_split's exact children (kdtree.py:441-467): tight boxes of slabs [0, k) and [k, e).
__device__ void sub_forced(const Span* __restrict__ sp, int e, int k, SubAxis& out) {
  const int lane = threadIdx.x & 31;
  RBox l = rb_empty(), r = rb_empty();
  for (int s = lane; s < e; s += 32) {
    if (s < k) l = rb_join(l, slab_box(sp, s));
    else r = rb_join(r, slab_box(sp, s));
  }
  l = rb_warp_reduce(l);
  r = rb_warp_reduce(r);
  if (lane == 0) { out.k = k; out.valid = 1; out.l = l; out.r = r; }
}

__device__ __forceinline__ Box sub_box(const SubEntry& e) {
  Box b;
  for (int k = 0; k < 3; ++k) { b.lo[k] = e.lo[k]; b.hi[k] = e.hi[k]; }
  return b;
}

__device__ __forceinline__ bool sub_push(SubSmem& sm, const Box& b, int parent, int depth,
                                         int right) {
  if (sm.sp >= SUB_STACK) return false;
  SubEntry e;
  for (int k = 0; k < 3; ++k) { e.lo[k] = (short)b.lo[k]; e.hi[k] = (short)b.hi[k]; }
  e.parent = parent;
  e.depth = (short)depth;
  e.right = (short)right;
  sm.stack[sm.sp++] = e;
  return true;
}

__global__ void __launch_bounds__(SUB_T) k_subtrees(const uint32_t* __restrict__ bits, int ny,
                                                    int nzw, KdParams P, SubCtx C) {
  extern __shared__ __align__(16) unsigned char sub_smem[];
  SubSmem& sm = *reinterpret_cast<SubSmem*>(sub_smem);
  uint32_t* words = reinterpret_cast<uint32_t*>(sub_smem + ((sizeof(SubSmem) + 15) & ~size_t(15)));
  const int t = threadIdx.x, warp = t >> 5;
  const int s = C.order ? C.order[blockIdx.x] : (int)blockIdx.x;
  const Box RB = C.rec[C.list[s]].box;
  const int exR = RB.hi[0] - RB.lo[0], eyR = RB.hi[1] - RB.lo[1], ezR = RB.hi[2] - RB.lo[2];
  const int wzR = (ezR + 31) >> 5;
  const int nw = exR * eyR * wzR;
  for (int q = t; q < nw; q += SUB_T) {
    const int w = q % wzR, rr = q / wzR, y = rr % eyR, x = rr / eyR;
    words[q] = local_word(bits + ((int64_t)(RB.lo[0] + x) * ny + RB.lo[1] + y) * nzw, RB.lo[2],
                          RB.hi[2], w);
  }
  if (t == 0) {
    Box root;
    for (int k = 0; k < 3; ++k) { root.lo[k] = 0; root.hi[k] = RB.hi[k] - RB.lo[k]; }
    sm.sp = 0;
    sub_push(sm, root, -1, 1, 0);
    sm.count = 0;
    sm.maxdepth = 0;
    sm.status = 0;
  }
  for (;;) {
    if (t == 0) {
      if (sm.sp == 0 || sm.status) sm.cur.depth = -1;
      else sm.cur = sm.stack[--sm.sp];
    }
    __syncthreads();
    const SubEntry e = sm.cur;
    if (e.depth < 0) break;
    const Box b = sub_box(e);
    const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
    const int64_t vol = box_vol(b);
    const bool sweep = !halted(P, vol);
    int fa = 0, fe = ex;
    if (ey > fe) { fa = 1; fe = ey; }
    if (ez > fe) { fa = 2; fe = ez; }
    const bool forced = P.mls >= 0 && fe > P.mls;
    if (sweep || forced) {
      sub_spans(sm, words, eyR, wzR, b);
      if (warp < 3) {
        const int a = warp;
        if (sweep)
          sub_sweep_axis(a == 0 ? sm.spx : (a == 1 ? sm.spy : sm.spz),
                         a == 0 ? ex : (a == 1 ? ey : ez), sm.ax[a]);
        else if ((t & 31) == 0)
          sm.ax[a].valid = 0;
      } else if (forced) {
        sub_forced(fa == 0 ? sm.spx : (fa == 1 ? sm.spy : sm.spz), fe, fe / 2, sm.forced);
      }
      __syncthreads();
    }
    if (t == 0) {
      int a = -1, k = 0;
      RBox l, r;
      if (sweep) {
        long long bc = 0;
        for (int q = 0; q < 3; ++q) {
          const SubAxis& A = sm.ax[q];
          if (!A.valid || (a >= 0 && A.cost >= bc)) continue;
          a = q; k = A.k; bc = A.cost; l = A.l; r = A.r;
        }
        if (a >= 0 && bc >= vol) a = -1;  // acceptance: cost < volume (kdtree.py:431, 436)
      }
      if (a < 0 && forced) { a = fa; k = sm.forced.k; l = sm.forced.l; r = sm.forced.r; }
      const int p = sm.count;
      bool ok = true;
      if ((p & (SUB_CHUNK - 1)) == 0) {
        const int ci = p / SUB_CHUNK;
        if (ci >= SUB_MAXCH) {
          sm.status |= 2;
          ok = false;
        } else {
          const unsigned long long c = atomicAdd(C.pool_used, 1ull);
          if ((long long)c >= C.pool_chunks) { sm.status |= 1; ok = false; }
          else sm.chunk[ci] = (int)c;
        }
      }
      if (ok) {
        sm.count = p + 1;
        sm.maxdepth = max(sm.maxdepth, (int)e.depth);
        SubRow* row = C.pool + (int64_t)sm.chunk[p / SUB_CHUNK] * SUB_CHUNK + (p & (SUB_CHUNK - 1));
        SubRow w;
        for (int q = 0; q < 3; ++q) { w.lo[q] = RB.lo[q] + b.lo[q]; w.hi[q] = RB.lo[q] + b.hi[q]; }
        w.axis = a;
        w.plane = a < 0 ? -1 : RB.lo[a] + (a == 0 ? b.lo[0] : (a == 1 ? b.lo[1] : b.lo[2])) + k;
        w.left = -1;
        w.right = -1;
        *row = w;
        if (e.parent >= 0) {
          SubRow* pr = C.pool + (int64_t)sm.chunk[e.parent / SUB_CHUNK] * SUB_CHUNK +
                       (e.parent & (SUB_CHUNK - 1));
          if (e.right) pr->right = p; else pr->left = p;
        }
        if (a >= 0) {  // right first: the left subtree is emitted next (DFS preorder)
          if (r.hi0 >= 0 && !sub_push(sm, to_global(b, a, r), p, e.depth + 1, 1)) sm.status |= 2;
          if (l.hi0 >= 0 && !sub_push(sm, to_global(b, a, l), p, e.depth + 1, 0)) sm.status |= 2;
        }
      }
    }
  }
  if (t == 0) {
    const int nch = (sm.count + SUB_CHUNK - 1) / SUB_CHUNK;
    sm.choff = (int)atomicAdd(C.chunks_used, (unsigned long long)nch);
    C.count[s] = sm.count;
    C.height[s] = sm.maxdepth;
    C.choff[s] = sm.choff;
    if (sm.status) atomicOr(C.status, sm.status);
  }
  __syncthreads();
  const int nch = (sm.count + SUB_CHUNK - 1) / SUB_CHUNK;
  for (int i = t; i < nch; i += SUB_T) C.chunks[sm.choff + i] = sm.chunk[i];
}

// Deferred records -> subtree ids (order irrelevant: every subtree is independent).
// Also sums a generous row-pool estimate (chunks: 1 + volume / 4096 per subtree).
__global__ void k_collect_sub(NodeRec* __restrict__ rec, int64_t total, int* __restrict__ list,
                              int64_t* __restrict__ nsub, int64_t* __restrict__ chunk_est) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total || rec[i].sub != SUB_DEFER) return;
  const int id = (int)atomicAdd(reinterpret_cast<unsigned long long*>(nsub), 1ull);
  rec[i].sub = id;
  list[id] = (int)i;
  atomicAdd(reinterpret_cast<unsigned long long*>(chunk_est),
            (unsigned long long)(1 + box_vol(rec[i].box) / 4096));
}

// The subtrees' launch order: by box volume (the work estimate) in power-of-two classes,
// biggest class first, so the big subtrees start first and the small ones fill in behind
// them (LPT-like order).  k_sub_class: class histogram; k_sub_order: each subtree's slot =
// its class offset (exclusive scan of the classes above, per block) + a slot counter.
constexpr int SUB_CLASSES = 32;
__device__ __forceinline__ int sub_class(const NodeRec* rec, const int* list, int64_t s) {
  const int64_t v = box_vol(rec[list[s]].box);
  return v > 0 ? 63 - __clzll(v) : 0;
}
__global__ void k_sub_class(const NodeRec* __restrict__ rec, const int* __restrict__ list,
                            int64_t nsub, int* __restrict__ hist) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nsub) atomicAdd(hist + sub_class(rec, list, s), 1);
}
__global__ void k_sub_order(const NodeRec* __restrict__ rec, const int* __restrict__ list,
                            int64_t nsub, const int* __restrict__ hist, int* __restrict__ cursor,
                            int* __restrict__ order) {
  __shared__ int off[SUB_CLASSES];
  if (threadIdx.x == 0) {
    int run = 0;
    for (int c = SUB_CLASSES - 1; c >= 0; --c) { off[c] = run; run += hist[c]; }
  }
  __syncthreads();
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsub) return;
  const int c = sub_class(rec, list, s);
  order[off[c] + atomicAdd(cursor + c, 1)] = (int)s;
}

// A subtree's rows at its global preorder p0 (the deferred record's), child links shifted.
__global__ void k_scatter_sub(const NodeRec* __restrict__ rec, const int* __restrict__ list,
                              SubCtx C, const int* __restrict__ pre, int32_t* __restrict__ lo,
                              int32_t* __restrict__ hi, int8_t* __restrict__ axis,
                              int32_t* __restrict__ plane, int32_t* __restrict__ left,
                              int32_t* __restrict__ right, int* __restrict__ height) {
  const int s = blockIdx.x;
  const int ri = list[s];
  const int p0 = pre[ri], cnt = C.count[s], off = C.choff[s];
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const SubRow w = C.pool[(int64_t)C.chunks[off + j / SUB_CHUNK] * SUB_CHUNK + (j & (SUB_CHUNK - 1))];
    const int p = p0 + j;
    for (int k = 0; k < 3; ++k) { lo[3 * p + k] = w.lo[k]; hi[3 * p + k] = w.hi[k]; }
    axis[p] = (int8_t)w.axis;
    plane[p] = w.plane;
    left[p] = w.left >= 0 ? p0 + w.left : -1;
    right[p] = w.right >= 0 ? p0 + w.right : -1;
  }
  if (threadIdx.x == 0) atomicMax(height, rec[ri].level + C.height[s]);
}

// ---- device-resident level loop (sweep builder) ---------------------------------------------
// The sweep tree's top is a long spine of big nodes (a cut often peels a thin slab off a node,
// so a 512^3 blob volume has ~75 levels of nodes too big for k_subtrees).  k_levels runs all
// those levels in ONE cooperative launch, two grid barriers per level:
//   phase A  every warp of the grid takes (node, slab, 64-row chunk) items of the level
//            (rows_or, as k_spans_rows) and merges x / y slab spans and the [w][slab] z-word
//            projections into the node's storage with atomics;
//   phase B  CTA per node: z-slab spans from the projections (ballots), the three sweeps
//            (block scans over a thread's run of slabs), acceptance / forced split, then the
//            children: rows (BFS records, level-ordered, slots by atomics), work entries for
//            the children that need a decision, their span / projection storage initialised.
// Leaves and deferred children (k_subtrees) get their record and no work entry.  Anything
// that does not fit the preallocated state (level width, records, storage, extents > 1024)
// aborts the launch and the host reruns the level-by-level path.
constexpr int LV_T = 256;
#ifndef VS_LV_U
#define VS_LV_U 8  // rows per lane in flight in phase A's vector loads
#endif
#ifndef VS_LV_TILED
#define VS_LV_TILED 0  // 1: phase A items in x/y band tiles (measured 2-3% slower; kept for A/B)
#endif
constexpr int LV_W = LV_T / 32;
constexpr int LV_NMAX = 1024;   // work nodes per level
constexpr int LV_EMAX = 1024;   // node extent per axis

struct LvNode {
  Box box;
  int rec;
  int sx, sy, sz;    // x / y slab spans (phase A) and z slab spans (phase B) in the span arena
  long long pz;      // [w][x] then [w][y] z-word projections in the level's word arena
};

struct LvCounters {
  int nwork[2];
  int nrec[2];       // records of the next level (by its parity)
  int abort;
  int nlevels;
  unsigned long long span_used[2];
  unsigned long long proj_used[2];
  long long total;
  long long root_vol;
};

struct LvCtx {
  const uint32_t* bits;
  int nx, ny, nz, nzw;
  KdParams P;
  const int* bbox;
  LvCounters* C;
  LvNode* work[2];
  NodeRec* rec;
  long long rec_cap;
  long long* level_base;
  int level_cap;
  Span* span[2];
  long long span_cap;
  uint32_t* proj[2];
  long long proj_cap;
  long long* prof;   // optional: %globaltimer at each phase boundary (3 per level)
  bool vec;          // packed rows 16-byte aligned (nzw % 4 == 0): phase A loads uint4
  struct LvAxisRes* res;  // 3 per work node
  int* arrive;            // per work node: axis CTAs done (reset by the deciding CTA)
  int* zarrive;           // per work node: z-column groups done (reset by the last one)
};

__device__ __forceinline__ long long lv_now() {
  long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

struct LvSmem {
  int off[LV_NMAX + 1];        // phase A: item offsets of the level's nodes
  Span stage[LV_EMAX];         // phase B: the axis' slab spans
  RBox suf[LV_EMAX];           // phase B: suffix boxes
  RBox wbox[LV_W];
  long long wcost[LV_W];
  int wk[LV_W];
  int wsum[LV_W];
  RBox best_l, best_r, ax_l[3], ax_r[3];
  long long ax_cost[3];
  int ax_k[3];
  int cnew[2];                 // work slots of the new children (-1 none)
  LvNode cnode[2];
  int last;
};

// Phase-A row geometry of a node: lanes per row (a lane group; 16-byte vectors when the
// packed rows allow it -- four z words per load) and rows per item (at most SPAN_CHUNK, two
// 8-deep load rounds).
struct LvGeom {
  int gwa, nwg, sh, wz;
  bool direct, vec;
  int v0, nv;   // vector path: first vector, vectors covering the node's stored words
  int gw, G, R;
};
__device__ __forceinline__ LvGeom lv_geom(const Box& b, bool vec_ok) {
  LvGeom q;
  q.gwa = b.lo[2] >> 5;
  q.sh = b.lo[2] & 31;
  q.nwg = ((b.hi[2] - 1) >> 5) - q.gwa + 1;
  q.wz = wz_of(b);
  q.direct = q.nwg <= 32;
  q.vec = q.direct && vec_ok;
  q.v0 = q.gwa >> 2;
  q.nv = ((q.gwa + q.nwg - 1) >> 2) - q.v0 + 1;
  q.gw = group_width(q.vec ? q.nv : (q.direct ? q.nwg : q.wz));
  q.G = 32 / q.gw;
  q.R = min(SPAN_CHUNK, 16 * q.G);
  return q;
}
__device__ __forceinline__ int lv_items(const Box& b, bool vec_ok) {
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], R = lv_geom(b, vec_ok).R;
  return ex * ((ey + R - 1) / R) + ey * ((ex + R - 1) / R);
}

// One slab's rows [r0, r1) with 16-byte loads: lane group of gw lanes per row, each lane one
// 4-word vector (masked to the node's stored words), U rows per lane in flight.
template <int U>
__device__ __forceinline__ void rows_or_v4(const uint32_t* __restrict__ bits, int ny, int nzw,
                                           int ax, int slab, int x0, int y0, int r0, int r1,
                                           int G, int g, int gw, uint32_t gmask, int vidx,
                                           uint4 m, uint4& acc, int& rmin, int& rmax) {
  for (int rb = r0; rb < r1; rb += G * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = min(rb + u * G + g, r1 - 1);
      const int x = ax == 0 ? slab : x0 + r;
      const int y = ax == 0 ? y0 + r : slab;
      v[u] = __ldg(reinterpret_cast<const uint4*>(bits + ((int64_t)x * ny + y) * nzw) + vidx);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = rb + u * G + g < r1;
      uint4 w;
      w.x = ok ? v[u].x & m.x : 0u;
      w.y = ok ? v[u].y & m.y : 0u;
      w.z = ok ? v[u].z & m.z : 0u;
      w.w = ok ? v[u].w & m.w : 0u;
      const uint32_t bm = __ballot_sync(0xffffffffu, (w.x | w.y | w.z | w.w) != 0);
      if ((bm >> (g * gw)) & gmask) {
        const int r = rb + u * G + g;
        rmin = min(rmin, r);
        rmax = max(rmax, r);
      }
      acc.x |= w.x; acc.y |= w.y; acc.z |= w.z; acc.w |= w.w;
    }
  }
}

__device__ __forceinline__ LvNode lv_load(const LvNode* p) {
  LvNode n;
  const int* s = reinterpret_cast<const int*>(p);
  int* d = reinterpret_cast<int*>(&n);
#pragma unroll
  for (int k = 0; k < (int)(sizeof(LvNode) / 4); ++k) d[k] = __ldcg(s + k);
  return n;
}
__device__ __forceinline__ Span lv_span(const Span* p) {
  const int4 v = __ldcg(reinterpret_cast<const int4*>(p));
  return Span{v.x, v.y, v.z, v.w};
}

// Block-wide exclusive scan of one int per thread (LV_T threads).
__device__ int lv_scan_int(int v, LvSmem& sm, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __syncthreads();
  if (lane == 31) sm.wsum[warp] = inc;
  __syncthreads();
  int before = 0;
  total = 0;
  for (int w = 0; w < LV_W; ++w) {
    if (w < warp) before += sm.wsum[w];
    total += sm.wsum[w];
  }
  return before + inc - v;
}

// ---- phase A: slab spans and projections of every node of the level ------------------------
__device__ void lv_phase_a(const LvCtx& X, const LvNode* __restrict__ work, int n, Span* spans,
                           uint32_t* proj, LvSmem& sm, long long* pf) {
  const int t = threadIdx.x, lane = t & 31;
  // item offsets (n <= LV_NMAX: NPT nodes per thread)
  constexpr int NPT = LV_NMAX / LV_T;
  int c[NPT], sum = 0;
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int i = NPT * t + j;
    c[j] = i < n ? lv_items(lv_load(work + i).box, X.vec) : 0;
    sum += c[j];
  }
  int total;
  int run = lv_scan_int(sum, sm, total);
#pragma unroll
  for (int j = 0; j < NPT; ++j) {
    const int i = NPT * t + j;
    if (i <= n) sm.off[i] = run;
    run += c[j];
  }
  if (t == 0) sm.off[n] = total;
  __syncthreads();
  if (pf) { pf[5] = lv_now(); pf[7] = total; }
  // a contiguous range of items per CTA, its warps striding through it: a warp's node
  // changes rarely (found by stepping forward, the node reloaded only then)
  const int chunk = (total + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * chunk, b1 = min(total, b0 + chunk);
  int node = -1;
  LvNode nd;
  for (int it = b0 + (t >> 5); it < b1; it += LV_W) {
    if (node < 0 || it >= sm.off[node + 1]) {
      if (node < 0) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.off[mid] <= it) lo = mid; else hi = mid - 1;
        }
        node = lo;
      } else {
        while (it >= sm.off[node + 1]) ++node;
      }
      nd = lv_load(work + node);
    }
    const Box b = nd.box;
    const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1];
    const LvGeom q = lv_geom(b, X.vec);
#if VS_LV_TILED
    // Items in (x band, y band) tiles of R x R rows: the tile's x-slab items (slabs of the x
    // band, rows = the y band) and its y-slab items (slabs of the y band, rows = the x band)
    // alternate, so the second read of a row is an L2 hit instead of a second DRAM pass.
    const int local = it - sm.off[node];
    const int R = q.R;
    const int chx = (ey + R - 1) / R, chy = (ex + R - 1) / R;
    const int rowfull = R * chx + ey;  // items of a full x band
    const int bx = min(local / rowfull, chy - 1);
    const int rem = local - bx * rowfull;
    const int nxb = min(R, ex - bx * R);
    const int by = min(rem / (nxb + R), chx - 1);
    const int j = rem - by * (nxb + R);
    const int nyb = min(R, ey - by * R), mxy = min(nxb, nyb);
    int AX, idx;
    if (j < 2 * mxy) {
      AX = j & 1; idx = j >> 1;
    } else {
      AX = nxb > nyb ? 0 : 1; idx = j - mxy;
    }
    const int s = AX == 0 ? bx * R + idx : by * R + idx;
    const int cc = AX == 0 ? by : bx;
#else
    int local = it - sm.off[node];
    const int chx = (ey + q.R - 1) / q.R, nxi = ex * chx;
    const int AX = local < nxi ? 0 : 1;
    if (AX) local -= nxi;
    const int nch = AX == 0 ? chx : (ex + q.R - 1) / q.R;
    const int s = local / nch, cc = local - s * nch;
#endif
    const int er = AX == 0 ? ey : ex, es = AX == 0 ? ex : ey;
    const int r0 = cc * q.R, r1 = min(er, r0 + q.R);
    const int wz = q.wz, sh = q.sh, gw = q.gw, G = q.G;
    const int g = lane / gw, wl = lane & (gw - 1);
    const uint32_t gmask = gw == 32 ? 0xffffffffu : ((1u << gw) - 1u);
    const int slab = b.lo[AX] + s;
    const int hb = b.hi[2] & 31;
    uint32_t acc = 0;
    int rmin = KD_FAR, rmax = -1;
    if (q.vec) {
      // lane wl loads vector v0 + wl: words 4(v0 + wl) .. +3, masked to [gwa, gwa + nwg)
      uint4 m;
      uint32_t mk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int w = 4 * (q.v0 + wl) + j;
        uint32_t mm = wl < q.nv && w >= q.gwa && w < q.gwa + q.nwg ? 0xffffffffu : 0u;
        if (w == q.gwa) mm &= 0xffffffffu << sh;
        if (w == q.gwa + q.nwg - 1 && hb) mm &= (1u << hb) - 1u;
        mk[j] = mm;
      }
      m.x = mk[0]; m.y = mk[1]; m.z = mk[2]; m.w = mk[3];
      uint4 a4 = make_uint4(0u, 0u, 0u, 0u);
      rows_or_v4<VS_LV_U>(X.bits, X.ny, X.nzw, AX, slab, b.lo[0], b.lo[1], r0, r1, G, g, gw, gmask,
                    q.v0 + min(wl, q.nv - 1), m, a4, rmin, rmax);
      for (int o = gw; o < 32; o <<= 1) {
        a4.x |= __shfl_xor_sync(0xffffffffu, a4.x, o);
        a4.y |= __shfl_xor_sync(0xffffffffu, a4.y, o);
        a4.z |= __shfl_xor_sync(0xffffffffu, a4.z, o);
        a4.w |= __shfl_xor_sync(0xffffffffu, a4.w, o);
        rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      }
      // stored words -> node-local word `lane`: (S[gwa+lane] >> sh) | (S[gwa+lane+1] << 32-sh)
      const int w1 = q.gwa + lane, w2 = w1 + 1;
      const int l1 = min(31, (w1 >> 2) - q.v0), l2 = min(31, (w2 >> 2) - q.v0);
      const uint32_t s1x = __shfl_sync(0xffffffffu, a4.x, l1), s1y = __shfl_sync(0xffffffffu, a4.y, l1);
      const uint32_t s1z = __shfl_sync(0xffffffffu, a4.z, l1), s1w = __shfl_sync(0xffffffffu, a4.w, l1);
      const uint32_t s2x = __shfl_sync(0xffffffffu, a4.x, l2), s2y = __shfl_sync(0xffffffffu, a4.y, l2);
      const uint32_t s2z = __shfl_sync(0xffffffffu, a4.z, l2), s2w = __shfl_sync(0xffffffffu, a4.w, l2);
      const int c1 = w1 & 3, c2 = w2 & 3;
      const uint32_t S1 = c1 == 0 ? s1x : (c1 == 1 ? s1y : (c1 == 2 ? s1z : s1w));
      const uint32_t S2 = c2 == 0 ? s2x : (c2 == 1 ? s2y : (c2 == 2 ? s2z : s2w));
      acc = lane < wz ? ((S1 >> sh) | (sh ? S2 << (32 - sh) : 0u)) : 0u;
    } else {
      int w0, w1;
      uint32_t wmask;
      if (q.direct) {
        w0 = w1 = q.gwa + min(wl, q.nwg - 1);
        wmask = wl < q.nwg ? 0xffffffffu : 0u;
        if (wl == 0) wmask &= 0xffffffffu << sh;
        if (wl == q.nwg - 1 && hb) wmask &= (1u << hb) - 1u;
      } else {
        const int wc = min(wl, wz - 1);
        const int gz = b.lo[2] + 32 * wc, rem = b.hi[2] - gz;
        w0 = gz >> 5;
        w1 = min(w0 + 1, X.nzw - 1);
        wmask = wl < wz ? (rem < 32 ? (1u << rem) - 1u : 0xffffffffu) : 0u;
      }
      if (q.direct)
        rows_or<8, true>(X.bits, X.ny, X.nzw, AX, slab, b.lo[0], b.lo[1], r0, r1, G, g, gw,
                         gmask, w0, w1, 0, wmask, acc, rmin, rmax);
      else
        rows_or<8, false>(X.bits, X.ny, X.nzw, AX, slab, b.lo[0], b.lo[1], r0, r1, G, g, gw,
                          gmask, w0, w1, sh, wmask, acc, rmin, rmax);
      for (int o = gw; o < 32; o <<= 1) {
        acc |= __shfl_xor_sync(0xffffffffu, acc, o);
        rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
      }
      if (q.direct) {  // stored words -> node-local words
        const uint32_t nx2 = __shfl_down_sync(0xffffffffu, acc, 1);
        if (sh) acc = (acc >> sh) | (wl + 1 < q.nwg ? nx2 << (32 - sh) : 0u);
        if (wl >= wz) acc = 0u;
      }
      if (lane >= gw) acc = 0u;  // one copy of the node-local words: lanes 0 .. wz-1
    }
    const uint32_t mz = __ballot_sync(0xffffffffu, acc != 0);
    if (rmax >= 0) {
      const int wf = __ffs(mz) - 1, wlst = 31 - __clz(mz);
      const uint32_t af = __shfl_sync(0xffffffffu, acc, wf), al = __shfl_sync(0xffffffffu, acc, wlst);
      Span* dst = spans + (AX == 0 ? nd.sx : nd.sy) + s;
      if (lane == 0) {
        atomicMin(&dst->mn1, rmin);
        atomicMax(&dst->mx1, rmax);
        atomicMin(&dst->mn2, 32 * wf + __ffs(af) - 1);
        atomicMax(&dst->mx2, 32 * wlst + 31 - __clz(al));
      }
      uint32_t* pdst = proj + nd.pz + (AX == 0 ? 0 : (long long)wz * ex) + s;
      if (lane < wz && acc) atomicOr(pdst + (long long)lane * es, acc);
    }
  }
  if (pf) {
    __syncthreads();
    if (t == 0) pf[6] = lv_now();
  }
}

// Exclusive block scan (join) of one box per thread in thread order or reverse order.
__device__ RBox lv_excl_scan(RBox x, bool rev, LvSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  RBox inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    const RBox u = rev ? rb_shfl_down(inc, o) : rb_shfl_up(inc, o);
    if (rev ? lane + o < 32 : lane >= o) inc = rb_join(inc, u);
  }
  RBox ex = rb_shfl(inc, rev ? min(lane + 1, 31) : max(lane - 1, 0));
  if (rev ? lane == 31 : lane == 0) ex = rb_empty();
  __syncthreads();
  if (rev ? lane == 0 : lane == 31) sm.wbox[warp] = inc;
  __syncthreads();
  for (int w = 0; w < LV_W; ++w)
    if (rev ? w > warp : w < warp) ex = rb_join(ex, sm.wbox[w]);
  return ex;
}

__device__ RBox lv_reduce(RBox r, LvSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  r = rb_warp_reduce(r);
  __syncthreads();
  if (lane == 0) sm.wbox[warp] = r;
  __syncthreads();
  RBox t = rb_empty();
  for (int w = 0; w < LV_W; ++w) t = rb_join(t, sm.wbox[w]);
  return t;
}

// _axis_sweep over sm.stage[0, e): first-minimum cut, its cost and boxes (sm.best_l / _r).
__device__ void lv_sweep(int e, LvSmem& sm, int& best_k, long long& best_cost) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (e + LV_T - 1) / LV_T;
  const int s0 = min(e, t * per), s1 = min(e, s0 + per);
  RBox loc = rb_empty();
  for (int s = s0; s < s1; ++s) loc = rb_join(loc, slab_box(sm.stage, s));
  RBox r = lv_excl_scan(loc, true, sm);
  for (int s = s1 - 1; s >= s0; --s) {
    r = rb_join(r, slab_box(sm.stage, s));
    sm.suf[s] = r;
  }
  RBox pre = lv_excl_scan(loc, false, sm);  // (its barriers publish suf)
  long long bc = LLONG_MAX;
  int bk = 0;
  RBox bpre = rb_empty();
  for (int s = s0; s < s1; ++s) {
    pre = rb_join(pre, slab_box(sm.stage, s));
    if (s + 1 < e) {
      const long long c = rvol(pre) + rvol(sm.suf[s + 1]);
      if (c < bc) { bc = c; bk = s + 1; bpre = pre; }
    }
  }
  const long long my_c = bc;
  const int my_k = bk;
  for (int o = 16; o; o >>= 1) {
    const long long c2 = __shfl_xor_sync(0xffffffffu, bc, o);
    const int k2 = __shfl_xor_sync(0xffffffffu, bk, o);
    if (c2 < bc || (c2 == bc && k2 < bk)) { bc = c2; bk = k2; }
  }
  __syncthreads();
  if (lane == 0) { sm.wcost[warp] = bc; sm.wk[warp] = bk; }
  __syncthreads();
  bc = sm.wcost[0];
  bk = sm.wk[0];
  for (int w = 1; w < LV_W; ++w)
    if (sm.wcost[w] < bc || (sm.wcost[w] == bc && sm.wk[w] < bk)) { bc = sm.wcost[w]; bk = sm.wk[w]; }
  if (my_c == bc && my_k == bk && bc != LLONG_MAX) { sm.best_l = bpre; sm.best_r = sm.suf[bk]; }
  __syncthreads();
  best_k = bk;
  best_cost = bc;
}

// Stage axis a's slab spans of node nd into sm.stage.
__device__ void lv_stage(const LvCtx& X, const Span* spans, const LvNode& nd, int a, int e,
                         LvSmem& sm) {
  __syncthreads();
  for (int s = threadIdx.x; s < e; s += LV_T)
    sm.stage[s] = lv_span(spans + (a == 0 ? nd.sx : (a == 1 ? nd.sy : nd.sz)) + s);
  __syncthreads();
}

// The children of a decided node (thread 0): records (level-ordered slots), and work entries
// for those that need a decision.  The four counter atomics are issued together (one L2 round
// trip), then consumed.
__device__ void lv_children(const LvCtx& X, const Box* cb, const bool* has, int level,
                            long long base_next, const KdParams& P, LvSmem& sm, int* rec_id) {
  LvCounters* C = X.C;
  const int nxt = (level + 1) & 1;
  bool work[2] = {false, false}, deferred[2] = {false, false};
  int nrec = 0, nwork = 0;
  unsigned long long nspan = 0, nproj = 0;
  for (int q = 0; q < 2; ++q) {
    rec_id[q] = -1;
    sm.cnew[q] = -1;
    if (!has[q]) continue;
    const Box& b = cb[q];
    const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
    const int mx = max(ex, max(ey, ez));
    const bool need = !halted(P, box_vol(b)) || (P.mls >= 0 && mx > P.mls);
    deferred[q] = need && defer_node(P, b);
    work[q] = need && !deferred[q];
    ++nrec;
    if (work[q]) {
      ++nwork;
      nspan += ex + ey + ez;
      nproj += ((unsigned long long)((ez + 31) >> 5) * (ex + ey) + 3) & ~3ull;
      if (mx > LV_EMAX) atomicExch(&C->abort, 1);
    }
  }
  if (!nrec) return;
  const int r0 = atomicAdd(&C->nrec[nxt], nrec);
  const int w0 = nwork ? atomicAdd(&C->nwork[nxt], nwork) : 0;
  const unsigned long long s0 = nwork ? atomicAdd(&C->span_used[nxt], nspan) : 0;
  const unsigned long long p0 = nwork ? atomicAdd(&C->proj_used[nxt], nproj) : 0;
  if (base_next + r0 + nrec > X.rec_cap || w0 + nwork > LV_NMAX ||
      (long long)(s0 + nspan) > X.span_cap || (long long)(p0 + nproj) > X.proj_cap) {
    atomicExch(&C->abort, 1);
    return;
  }
  int r = r0, w = w0;
  unsigned long long so = s0, po = p0;
  for (int q = 0; q < 2; ++q) {
    if (!has[q]) continue;
    const Box& b = cb[q];
    const long long rid = base_next + r++;
    rec_id[q] = (int)rid;
    NodeRec rr;
    rr.box = b;
    rr.axis = -1; rr.plane = -1; rr.left = -1; rr.right = -1; rr.dropped = 0;
    rr.level = level + 1;
    rr.sub = deferred[q] ? SUB_DEFER : -1;
    X.rec[rid] = rr;
    if (!work[q]) continue;
    const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
    LvNode nd;
    nd.box = b;
    nd.rec = (int)rid;
    nd.sx = (int)so;
    nd.sy = (int)(so + ex);
    nd.sz = (int)(so + ex + ey);
    nd.pz = (long long)po;
    so += ex + ey + ez;
    po += ((unsigned long long)wz_of(b) * (ex + ey) + 3) & ~3ull;
    X.work[nxt][w] = nd;
    sm.cnew[q] = w++;
    sm.cnode[q] = nd;
  }
}

// Empty spans / zero projections for a new work node (the whole CTA).
__device__ void lv_init_storage(const LvCtx& X, const LvNode& nd, int nxt) {
  const Box& b = nd.box;
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], wz = wz_of(b);
  int4* sp = reinterpret_cast<int4*>(X.span[nxt] + nd.sx);
  for (int i = threadIdx.x; i < ex + ey; i += LV_T) sp[i] = make_int4(KD_FAR, -1, KD_FAR, -1);
  // projection blocks start 16-byte aligned (lv_children rounds them to 4 words)
  uint4* pw = reinterpret_cast<uint4*>(X.proj[nxt] + nd.pz);
  const long long nw = ((long long)wz * (ex + ey) + 3) >> 2;
  for (long long i = threadIdx.x; i < nw; i += LV_T) pw[i] = make_uint4(0u, 0u, 0u, 0u);
}

// ---- phase B: node decisions, one CTA per (node, axis) -------------------------------------
// Each axis' sweep (and the forced split's boxes on the longest axis) runs on its own CTA and
// is published to lv_res; the last of a node's three CTAs to arrive (arrival counter) decides
// the node and creates its children -- the three sweeps run in parallel.
struct LvAxisRes {
  long long cost;
  int k, valid, fvalid, pad;
  RBox l, r, fl, fr;
};

// z-slab spans of node nd, columns [g*LV_W, g*LV_W + LV_W) of its 2*wz (axis, z word)
// columns, one warp each: first / last x (y) whose projection word holds each z bit, into the
// node's global z spans (x columns write mn1/mx1, y columns mn2/mx2; every field of every z
// slab is written by exactly one column).  The [w][slab] column (<= 1024 slabs) is held in
// registers, one word per lane per 32-slab chunk, and bit-transposed chunk by chunk.
__device__ void lv_zcolumns(const uint32_t* __restrict__ proj, Span* __restrict__ zs,
                            const LvNode& nd, int g, int kc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Box& b = nd.box;
  const int ex = b.hi[0] - b.lo[0], ey = b.hi[1] - b.lo[1], ez = b.hi[2] - b.lo[2];
  const int wz = (ez + 31) >> 5;
  for (int col = (g * LV_W + warp) * kc; col < min(2 * wz, (g * LV_W + warp + 1) * kc); ++col) {
  const bool isx = col < wz;
  const int w = isx ? col : col - wz;
  const int e = isx ? ex : ey, nch = (e + 31) >> 5;
  const uint32_t* p = proj + nd.pz + (isx ? 0 : (long long)wz * ex) + (long long)w * e;
  uint32_t v[LV_EMAX / 32];
#pragma unroll
  for (int c = 0; c < LV_EMAX / 32; ++c) {
    const int idx = c * 32 + lane;
    v[c] = c < nch && idx < e ? __ldcg(p + idx) : 0u;
  }
  int first = KD_FAR, last = -1;
#pragma unroll
  for (int c = 0; c < LV_EMAX / 32; ++c) {
    if (c < nch) {
      uint32_t x = v[c];
#pragma unroll
      for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t m = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu
                           : j == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
      }
      if (x) {
        if (first == KD_FAR) first = 32 * c + __ffs(x) - 1;
        last = 32 * c + 31 - __clz(x);
      }
    }
  }
  const int z = 32 * w + lane;
  if (z < ez) {
    int* d = reinterpret_cast<int*>(zs + nd.sz + z) + (isx ? 0 : 2);
    d[0] = first;
    d[1] = last;
  }
  }  // columns of the warp
}

// z-column groups of a node (kc columns per warp, LV_W warps; one group even when z needs no
// spans); kc is chosen per level so that the level's phase-B tasks fit the grid.
__device__ __forceinline__ int lv_zgroups(const Box& b, int kc) {
  const int wz = (b.hi[2] - b.lo[2] + 31) >> 5;
  return (2 * wz + LV_W * kc - 1) / (LV_W * kc);
}

struct LvNodeInfo {
  int ex, ey, ez, fa, fe;
  bool sweep, forced;
  int64_t vol;
};
__device__ __forceinline__ LvNodeInfo lv_info(const KdParams& P, const Box& b) {
  LvNodeInfo f;
  f.ex = b.hi[0] - b.lo[0]; f.ey = b.hi[1] - b.lo[1]; f.ez = b.hi[2] - b.lo[2];
  f.fa = 0; f.fe = f.ex;
  if (f.ey > f.fe) { f.fa = 1; f.fe = f.ey; }
  if (f.ez > f.fe) { f.fa = 2; f.fe = f.ez; }
  f.vol = box_vol(b);
  f.sweep = !halted(P, f.vol);
  f.forced = P.mls >= 0 && f.fe > P.mls;
  return f;
}

__device__ void lv_finish(const LvCtx& X, const KdParams& P, const LvNode& nd, int i, int level,
                          long long base_next, LvSmem& sm);
__device__ void lv_axis(const LvCtx& X, const KdParams& P, const LvNode& nd, int i, int a,
                        int level, long long base_next, LvSmem& sm);

// Phase-B task q of node i: 0 / 1 the x / y sweep, 2.. the z-column groups; the last group
// to finish runs the z sweep (lv_axis(2)) from the completed z spans.
__device__ void lv_task(const LvCtx& X, const KdParams& P, const LvNode& nd, int i, int q,
                        int kc, int level, long long base_next, LvSmem& sm) {
  if (q < 2) {
    lv_axis(X, P, nd, i, q, level, base_next, sm);
    return;
  }
  const int cur = level & 1;
  const LvNodeInfo f = lv_info(P, nd.box);
  const bool need_z = (f.sweep && f.ez >= 2) || (f.forced && f.fa == 2);
  if (need_z) lv_zcolumns(X.proj[cur], X.span[cur], nd, q - 2, kc);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int ng = lv_zgroups(nd.box, kc);
    const int prev = atomicAdd(X.zarrive + i, 1);
    sm.last = prev == ng - 1;
    if (sm.last) X.zarrive[i] = 0;
  }
  __syncthreads();
  if (sm.last) {
    __threadfence();
    lv_axis(X, P, nd, i, 2, level, base_next, sm);
  }
}

// Axis a of node i (work-list index): its sweep and, on the longest axis, the forced boxes.
__device__ void lv_axis(const LvCtx& X, const KdParams& P, const LvNode& nd, int i, int a,
                        int level, long long base_next, LvSmem& sm) {
  const int t = threadIdx.x;
  const int cur = level & 1;
  const LvNodeInfo f = lv_info(P, nd.box);
  const int e = a == 0 ? f.ex : (a == 1 ? f.ey : f.ez);
  const bool do_sweep = f.sweep && e >= 2, do_forced = f.forced && a == f.fa;
  LvAxisRes* res = X.res + 3 * i + a;
  if (do_sweep || do_forced) {
    lv_stage(X, X.span[cur], nd, a, e, sm);
    if (do_sweep) {
      int k;
      long long c;
      lv_sweep(e, sm, k, c);
      if (t == 0) { res->cost = c; res->k = k; res->l = sm.best_l; res->r = sm.best_r; }
    }
    if (do_forced) {
      const int k = e / 2;
      RBox lp = rb_empty(), rp = rb_empty();
      for (int s = t; s < e; s += LV_T) {
        if (s < k) lp = rb_join(lp, slab_box(sm.stage, s));
        else rp = rb_join(rp, slab_box(sm.stage, s));
      }
      const RBox l = lv_reduce(lp, sm), r = lv_reduce(rp, sm);
      if (t == 0) { res->fl = l; res->fr = r; }
    }
  }
  if (t == 0) {
    res->valid = do_sweep;
    res->fvalid = do_forced;
    if (X.prof && i == 0 && level < 1000) X.prof[16000 + 4 * level + a] = lv_now();
    __threadfence();
    sm.last = atomicAdd(X.arrive + i, 1) == 2;
  }
  __syncthreads();
  if (sm.last) lv_finish(X, P, nd, i, level, base_next, sm);
  __syncthreads();
  if (sm.last && X.prof && i == 0 && t == 0 && level < 1000) X.prof[16000 + 4 * level + 3] = lv_now();
}

// The node's decision from its three axis results, its children and their storage.
__device__ void lv_finish(const LvCtx& X, const KdParams& P, const LvNode& nd, int i, int level,
                          long long base_next, LvSmem& sm) {
  const int t = threadIdx.x;
  const Box b = nd.box;
  if (t == 0) {
    __threadfence();
    const LvNodeInfo f = lv_info(P, b);
    // the three axis results in one round of independent L2 loads
    constexpr int RW = sizeof(LvAxisRes) / 4;
    int rw[3][RW];
    const int* src = reinterpret_cast<const int*>(X.res + 3 * i);
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int j = 0; j < RW; ++j) rw[q][j] = __ldcg(src + q * RW + j);
    const LvAxisRes* res = reinterpret_cast<const LvAxisRes*>(&rw[0][0]);
    int a = -1, k = 0;
    long long bc = 0;
    RBox l, r;
    if (f.sweep) {
      for (int q = 0; q < 3; ++q) {
        if (!res[q].valid || (a >= 0 && res[q].cost >= bc)) continue;
        a = q; bc = res[q].cost; k = res[q].k; l = res[q].l; r = res[q].r;
      }
      if (a >= 0 && bc >= f.vol) a = -1;  // acceptance: cost < volume (kdtree.py:431, 436)
    }
    if (a < 0 && f.forced) {
      a = f.fa;
      k = f.fe / 2;
      l = res[a].fl;
      r = res[a].fr;
    }
    NodeRec me;
    me.box = b;
    me.axis = a;
    me.plane = a < 0 ? -1 : (a == 0 ? b.lo[0] : (a == 1 ? b.lo[1] : b.lo[2])) + k;
    me.left = me.right = -1;
    me.dropped = 0;
    me.level = level;
    me.sub = -1;
    sm.cnew[0] = sm.cnew[1] = -1;
    if (a >= 0) {
      Box cb[2];
      bool has[2] = {l.hi0 >= 0, r.hi0 >= 0};
      if (has[0]) cb[0] = to_global(b, a, l);
      if (has[1]) cb[1] = to_global(b, a, r);
      int rid[2];
      lv_children(X, cb, has, level, base_next, P, sm, rid);
      me.left = rid[0];
      me.right = rid[1];
    }
    X.rec[nd.rec] = me;
    X.arrive[i] = 0;
  }
  __syncthreads();
  const int nxt = (level + 1) & 1;
  for (int q = 0; q < 2; ++q)
    if (sm.cnew[q] >= 0) lv_init_storage(X, sm.cnode[q], nxt);
}

#ifndef VS_LV_MINB
#define VS_LV_MINB 2
#endif
__global__ void __launch_bounds__(LV_T, VS_LV_MINB) k_levels(LvCtx X) {
  extern __shared__ __align__(16) unsigned char lv_smem[];
  LvSmem& sm = *reinterpret_cast<LvSmem*>(lv_smem);
  cg::grid_group grid = cg::this_grid();
  LvCounters* C = X.C;
  const int t = threadIdx.x;
  // root (kdtree.py:398): the bbox of every flag
  Box root;
  int bb[6];
  for (int q = 0; q < 6; ++q) bb[q] = __ldcg(X.bbox + q);
  for (int q = 0; q < 3; ++q) { root.lo[q] = bb[q]; root.hi[q] = bb[3 + q]; }
  if (bb[3] < 0) {  // empty volume
    if (blockIdx.x == 0 && t == 0) { C->nlevels = 0; C->total = 0; }
    return;
  }
  KdParams P = X.P;
  P.root_vol = box_vol(root);
  {
    const int ex = root.hi[0] - root.lo[0], ey = root.hi[1] - root.lo[1], ez = root.hi[2] - root.lo[2];
    const int mx = max(ex, max(ey, ez));
    const bool need = !halted(P, P.root_vol) || (P.mls >= 0 && mx > P.mls);
    const bool deferred = need && defer_node(P, root);
    const bool work = need && !deferred;
    const int wz = (ez + 31) >> 5;
    if (blockIdx.x == 0 && t == 0) {
      NodeRec r;
      r.box = root;
      r.axis = r.plane = r.left = r.right = -1;
      r.dropped = 0;
      r.level = 0;
      r.sub = deferred ? SUB_DEFER : -1;
      X.rec[0] = r;
      X.level_base[0] = 0;
      C->nwork[0] = work ? 1 : 0;
      if (work) {
        if (mx > LV_EMAX) C->abort = 1;
        LvNode nd;
        nd.box = root; nd.rec = 0; nd.sx = 0; nd.sy = ex; nd.sz = ex + ey; nd.pz = 0;
        X.work[0][0] = nd;
      }
    }
    if (work) {  // root storage, grid-stride
      const long long nspan = ex + ey + ez, nw = (long long)wz * (ex + ey);
      const long long g0 = (long long)blockIdx.x * LV_T + t, gs = (long long)gridDim.x * LV_T;
      for (long long i = g0; i < nspan; i += gs) X.span[0][i] = Span{KD_FAR, -1, KD_FAR, -1};
      for (long long i = g0; i < nw; i += gs) X.proj[0][i] = 0u;
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && t == 0) C->root_vol = P.root_vol;
  long long base = 0, nrec = 1;
  int level = 0;
  for (;;) {
    if (X.prof && blockIdx.x == 0 && t == 0 && level < 1000) X.prof[3 * level] = lv_now();
    const int cur = level & 1, nxt = cur ^ 1;
    const int n = *(volatile int*)&C->nwork[cur];
    if (n == 0 || *(volatile int*)&C->abort) break;
    if (blockIdx.x == 0 && t == 0) {
      C->nwork[nxt] = 0;
      C->nrec[nxt] = 0;
      C->span_used[nxt] = 0;
      C->proj_used[nxt] = 0;
    }
    lv_phase_a(X, X.work[cur], n, X.span[cur], X.proj[cur], sm,
               X.prof && blockIdx.x == 0 && level < 1000 ? X.prof + 3000 + 8 * level : nullptr);
    grid.sync();
    if (X.prof && blockIdx.x == 0 && t == 0 && level < 1000) X.prof[3 * level + 1] = lv_now();
    {
      // task offsets: 2 + z-column groups per node (every CTA scans them itself); columns per
      // warp kc so that the tasks fit the grid
      constexpr int NPT = LV_NMAX / LV_T;
      int c[NPT], wzs[NPT], sum = 0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int i = NPT * t + j;
        wzs[j] = 0;
        if (i < n) {
          const LvNode* w = X.work[cur] + i;
          wzs[j] = (__ldcg(&w->box.hi[2]) - __ldcg(&w->box.lo[2]) + 31) >> 5;
          sum += 2 * wzs[j];
        }
      }
      int total;
      lv_scan_int(sum, sm, total);  // total z columns of the level
      const int spare = max((int)gridDim.x - 2 * n, n);
      const int kc = max(1, (total + spare * LV_W - 1) / (spare * LV_W));
      sum = 0;
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int i = NPT * t + j;
        c[j] = i < n ? 2 + (2 * wzs[j] + LV_W * kc - 1) / (LV_W * kc) : 0;
        sum += c[j];
      }
      int run = lv_scan_int(sum, sm, total);
#pragma unroll
      for (int j = 0; j < NPT; ++j) {
        const int i = NPT * t + j;
        if (i <= n) sm.off[i] = run;
        run += c[j];
      }
      __syncthreads();
      int i = 0;
      for (int task = blockIdx.x; task < total; task += gridDim.x) {
        while (task >= sm.off[i + 1]) ++i;
        const LvNode nd = lv_load(X.work[cur] + i);
        lv_task(X, P, nd, i, task - sm.off[i], kc, level, base + nrec, sm);
        __syncthreads();
      }
    }
    grid.sync();
    if (X.prof && blockIdx.x == 0 && t == 0 && level < 1000) X.prof[3 * level + 2] = lv_now();
    const long long nn = *(volatile int*)&C->nrec[nxt];
    base += nrec;
    nrec = nn;
    ++level;
    if (level + 1 >= X.level_cap) {
      if (blockIdx.x == 0 && t == 0) C->abort = 1;
      break;
    }
    if (blockIdx.x == 0 && t == 0) X.level_base[level] = base;
  }
  if (blockIdx.x == 0 && t == 0 && !*(volatile int*)&C->abort) {
    const int nl = nrec > 0 ? level + 1 : level;
    C->nlevels = nl;
    C->total = base + nrec;
    X.level_base[nl] = base + nrec;
  }
}

}  // namespace vs

using namespace vs;

namespace {

// The library's stream-ordered pool: freed scratch stays mapped (release threshold = max), so
// a build's per-level buffers and the next build's reuse them without remapping memory.
cudaMemPool_t lib_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> g(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceGetDefaultMemPool(&pool, dev);
  }
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  pools[dev] = pool;
  return pool;
}

// Grow-only stream-ordered scratch buffer (data-dependent sizes: the k-d tree's level widths
// are only known as it is built).
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaStream_t st = nullptr;
  int ensure(size_t bytes, const char* what) {
    if (bytes <= cap) return 0;
    if (p) cudaFreeAsync(p, st);
    size_t nb = std::max(bytes, cap * 3 / 2 + 256);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaMallocFromPoolAsync(&p, nb, lib_pool(dev), st);
    if (e != cudaSuccess) {
      p = nullptr;
      cap = 0;
      set_error("%s: cudaMallocFromPoolAsync(%zu): %s", what, nb, cudaGetErrorString(e));
      return (int)e;
    }
    cap = nb;
    return 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  ~DBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

struct KdResultImpl {
  int64_t m = 0;
  int root = -1;
  int height = 0;
  DBuf lo, hi, axis, plane, left, right;
};

// Small device -> host reads (the level loop's per-level header) go through a per-thread
// pinned staging buffer: a pageable copy is staged by the driver and costs a few us more.
int d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
  constexpr size_t STAGE = 64 << 10;
  thread_local void* stage = nullptr;
  if (n <= STAGE && !stage && cudaMallocHost(&stage, STAGE) != cudaSuccess) {
    cudaGetLastError();
    stage = nullptr;
  }
  const bool pinned = n <= STAGE && stage;
  VS_CUDA(cudaMemcpyAsync(pinned ? stage : dst, src, n, cudaMemcpyDeviceToHost, st), "d2h");
  VS_CUDA(cudaStreamSynchronize(st), "sync");
  if (pinned) memcpy(dst, stage, n);
  return 0;
}

constexpr int SPAN_BLOCKS = 148 * 8;
#ifndef VS_ORDER_GRID
#define VS_ORDER_GRID 1  // trees > VS_ORDER_GRID_MIN rows: preorder passes over a cooperative grid
#endif
#ifndef VS_ORDER_GRID_MIN
#define VS_ORDER_GRID_MIN 65536
#endif
#ifndef VS_SUB_LPT
#define VS_SUB_LPT 1  // k_subtrees launched biggest subtree first (0: in collection order)
#endif
#ifndef VS_BINNED_WPN
#define VS_BINNED_WPN 8  // warps per node on narrow levels
#endif
#ifndef VS_BINNED_NARROW
#define VS_BINNED_NARROW 1024  // levels of at most this many nodes: 8 warps per node decision
#endif
constexpr int BINNED_NARROW = VS_BINNED_NARROW;

// A non-blocking side stream per device for independent passes (created once).
cudaStream_t side_stream(int dev) {
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  std::lock_guard<std::mutex> g(mu);
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  streams[dev] = s;
  return s;
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  int create() {
    VS_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
    VS_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
    return 0;
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

unsigned grid_for(int64_t items, int per_block, int cap = 148 * 64) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(items, per_block), cap));
}

}  // namespace

namespace {

constexpr int KD_RETRY_LEVELS = 1000;  // a subtree outgrew one CTA: rebuild level by level

// Level-synchronous build with one host synchronisation per level: the level's work sizes
// are computed where its boxes are emitted (prep_node) and scanned on the device; the host
// reads {node count, totals} once, sizes the level's buffers and launches the span passes,
// the decisions and the next level's emission.  Nodes small enough for one CTA leave the
// level loop (sweep builder) and are finished by k_subtrees.
int kd_build(const uint32_t* bits, int nx, int ny, int nz, int deep, int mls, int binned,
             int bins, int cs, const int* bbox_in, int subtrees, int dev_levels,
             KdResultImpl* R, cudaStream_t st) {
  const int nzw = (int)nzw_of(nz);

  DBuf bb, cur, nxt, offs, dec, cnt, spx, spy, spz, pxz, pyz, scr, rec, cellb, cpk, cslab, sizes,
      pre, hdr;
  for (DBuf* b : {&bb, &cur, &nxt, &offs, &dec, &cnt, &spx, &spy, &spz, &pxz, &pyz, &scr, &rec,
                  &cellb, &cpk, &cslab, &sizes, &pre, &hdr})
    b->st = st;

  KdParams P;
  P.deep = deep; P.mls = mls; P.binned = binned; P.bins = bins; P.cs = cs; P.root_vol = 0;
  P.subtrees = subtrees && !binned;
  const int ncx = (int)cdiv(nx, cs), ncy = (int)cdiv(ny, cs), ncz = (int)cdiv(nz, cs);
  // side stream (per device, cached) + fork/join events for the concurrent span passes
  int dev = 0;
  VS_CUDA(cudaGetDevice(&dev), "device");
  cudaStream_t side = side_stream(dev);
  if (!side) { set_error("vs_kd_build: side stream"); return VS_EINVAL; }
  EventPair evs;
  VS_TRY(evs.create());
  cudaEvent_t ev_fork = evs.a, ev_join = evs.b;

  // header: [0] node count of the level being prepared, [1 + k] total of offset array k,
  // [KA + 1] child total (next level's node count), [KA + 2 ..] root bbox ints
  constexpr int H = KA + 4;
  VS_TRY(hdr.ensure(H * sizeof(int64_t) + 8 * sizeof(int), "header"));
  int64_t* dh = hdr.as<int64_t>();
  int* dbb = reinterpret_cast<int*>(dh + H);
  int64_t hh[H];

  // per-level offset arrays: KA arrays of stride cap + 1
  int64_t cap = 0;
  auto arrays = [&](int64_t need_cap) -> int {
    if (need_cap > cap) {
      cap = std::max<int64_t>(need_cap, cap * 2);
      VS_TRY(offs.ensure((size_t)KA * (cap + 1) * sizeof(int64_t), "offsets"));
    }
    return 0;
  };
  auto arr = [&](int k) { return offs.as<int64_t>() + (int64_t)k * (cap + 1); };
  auto prep_ctx = [&]() {
    PrepCtx C;
    C.P = P;
    C.nc[0] = ncx; C.nc[1] = ncy; C.nc[2] = ncz;
    for (int k = 0; k < KA; ++k) C.arr[k] = arr(k);
    return C;
  };
  const int nscan = binned ? 6 : A_IZ + 1;
  const int scan0 = binned ? A_C0 : 0;
  DBuf part;
  part.st = st;
  // exclusive scans of S's arrays of n entries (n_dev on the device, else n_host); n_bound:
  // the host's bound on n.  Narrow: one block per array; wide: tiles across blocks.
  auto scan_arrays = [&](const ScanSet& S, const int64_t* n_dev, int64_t n_host,
                         int64_t n_bound) -> int {
    const int64_t nch = cdiv(std::max<int64_t>(n_bound, 1), SCAN_TILE);
    if (nch <= 2) {
      k_multi_scan<<<S.k, 1024, 0, st>>>(S, n_dev, n_host);
      return check_launch("k_multi_scan");
    }
    VS_TRY(part.ensure((size_t)S.k * nch * sizeof(int64_t), "scan partials"));
    const dim3 g((unsigned)nch, (unsigned)S.k);
    k_scan_sums<<<g, 256, 0, st>>>(S, n_dev, n_host, part.as<int64_t>(), (int)nch);
    VS_TRY(check_launch("k_scan_sums"));
    k_scan_apply<<<g, 1024, 0, st>>>(S, n_dev, n_host, part.as<int64_t>(), (int)nch);
    return check_launch("k_scan_apply");
  };
  auto scan_level = [&](const int64_t* n_dev, int64_t n_bound) -> int {
    ScanSet S;
    S.k = nscan;
    for (int j = 0; j < nscan; ++j) {
      S.a[j] = arr(scan0 + j);
      S.totals[j] = dh + 1 + scan0 + j;
    }
    return scan_arrays(S, n_dev, 0, n_bound);
  };

  // root box (kdtree.py:398): tight box of every flag
  const int init[8] = {KD_FAR, KD_FAR, KD_FAR, -1, -1, -1, 0, 0};
  VS_CUDA(cudaMemcpyAsync(dbb, init, sizeof init, cudaMemcpyHostToDevice, st), "bbox init");
  VS_CUDA(cudaMemsetAsync(dh, 0, H * sizeof(int64_t), st), "header init");
  if (bbox_in) {  // the root box came with the bits (k_classify_pack)
    VS_CUDA(cudaMemcpyAsync(dbb, bbox_in, 6 * sizeof(int), cudaMemcpyDeviceToDevice, st),
            "bbox copy");
  } else {
    k_bits_bbox<<<SPAN_BLOCKS, 256, 0, st>>>(bits, nx, ny, nz, dbb);
    VS_TRY(check_launch("k_bits_bbox"));
  }
  std::vector<int64_t> level_base;
  int64_t total = -1;
  DBuf lv_work, lv_ctr, lv_lb, lv_span, lv_proj, lv_res;
  for (DBuf* b : {&lv_work, &lv_ctr, &lv_lb, &lv_span, &lv_proj, &lv_res}) b->st = st;
  if (P.subtrees && dev_levels && nx <= LV_EMAX && ny <= LV_EMAX && nz <= LV_EMAX) {
    // the whole big-node part of the tree in one cooperative launch (k_levels)
    const long long rec_cap = 1 << 18, span_cap = 2LL * LV_NMAX * LV_EMAX;
    const long long proj_cap = std::max<long long>(4LL << 20, (long long)nx * ny * nzw / 4);
    const int level_cap = 4096;
    VS_TRY(rec.ensure(rec_cap * sizeof(NodeRec), "records"));
    VS_TRY(lv_work.ensure(2 * LV_NMAX * sizeof(LvNode), "level work"));
    VS_TRY(lv_ctr.ensure(sizeof(LvCounters), "level counters"));
    VS_TRY(lv_lb.ensure(level_cap * sizeof(long long), "level bases"));
    VS_TRY(lv_span.ensure(2 * span_cap * sizeof(Span), "level spans"));
    VS_TRY(lv_proj.ensure(2 * proj_cap * sizeof(uint32_t), "level projections"));
    VS_CUDA(cudaMemsetAsync(lv_ctr.p, 0, sizeof(LvCounters), st), "level counters");
    const size_t res_bytes = 3 * LV_NMAX * sizeof(LvAxisRes);
    VS_TRY(lv_res.ensure(res_bytes + 2 * LV_NMAX * sizeof(int), "axis results"));
    VS_CUDA(cudaMemsetAsync(static_cast<char*>(lv_res.p) + res_bytes, 0,
                            2 * LV_NMAX * sizeof(int), st), "arrivals");
    LvCtx X;
    X.bits = bits; X.nx = nx; X.ny = ny; X.nz = nz; X.nzw = nzw;
    X.P = P;
    X.bbox = dbb;
    X.C = lv_ctr.as<LvCounters>();
    X.work[0] = lv_work.as<LvNode>();
    X.work[1] = lv_work.as<LvNode>() + LV_NMAX;
    X.rec = rec.as<NodeRec>();
    X.rec_cap = rec_cap;
    X.level_base = lv_lb.as<long long>();
    X.level_cap = level_cap;
    X.span[0] = lv_span.as<Span>();
    X.span[1] = lv_span.as<Span>() + span_cap;
    X.span_cap = span_cap;
    X.proj[0] = lv_proj.as<uint32_t>();
    X.proj[1] = lv_proj.as<uint32_t>() + proj_cap;
    X.proj_cap = proj_cap;
    X.prof = nullptr;
    X.vec = (nzw & 3) == 0 && ((uintptr_t)bits & 15) == 0;
    X.res = lv_res.as<LvAxisRes>();
    X.arrive = reinterpret_cast<int*>(static_cast<char*>(lv_res.p) + res_bytes);
    X.zarrive = X.arrive + LV_NMAX;
    DBuf lv_prof;
    lv_prof.st = st;
    const char* penv = getenv("VSB200_KD_PROFILE");
    if (penv && penv[0] == '1') {
      VS_TRY(lv_prof.ensure(20000 * sizeof(long long), "profile"));
      VS_CUDA(cudaMemsetAsync(lv_prof.p, 0, 20000 * sizeof(long long), st), "profile");
      X.prof = lv_prof.as<long long>();
    }
    const size_t smem = sizeof(LvSmem);
    VS_CUDA(cudaFuncSetAttribute(k_levels, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "k_levels smem");
    int per_sm = 0, nsm = 0;
    VS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels, LV_T, smem),
            "k_levels occupancy");
    VS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "SM count");
    if (per_sm > 0) {
      void* args[] = {&X};
      VS_CUDA(cudaLaunchCooperativeKernel((void*)k_levels, dim3(nsm * per_sm), dim3(LV_T), args,
                                          smem, st), "k_levels");
      LvCounters hc;
      VS_TRY(d2h(&hc, lv_ctr.p, sizeof hc, st));
      if (X.prof) {  // dev profile: per-phase sums over the levels
        std::vector<long long> pr(20000);
        VS_TRY(d2h(pr.data(), X.prof, pr.size() * sizeof(long long), st));
        for (int l = 0; l < std::min(hc.nlevels - 1, 12); ++l)
          fprintf(stderr, "  level %d node 0 axis done x %.1f y %.1f z %.1f finish %.1f us\n", l,
                  (pr[16000 + 4 * l] - pr[3 * l + 1]) * 1e-3, (pr[16001 + 4 * l] - pr[3 * l + 1]) * 1e-3,
                  (pr[16002 + 4 * l] - pr[3 * l + 1]) * 1e-3, (pr[16003 + 4 * l] - pr[3 * l + 1]) * 1e-3);
        for (int l = 0; l < std::min(hc.nlevels - 1, 12); ++l)
          fprintf(stderr, "  level %d: A scan %.1f block0 %.1f all %.1f us (%lld items) | B %.1f us\n",
                  l, (pr[3000 + 8 * l + 5] - pr[3 * l]) * 1e-3,
                  (pr[3000 + 8 * l + 6] - pr[3 * l]) * 1e-3, (pr[3 * l + 1] - pr[3 * l]) * 1e-3,
                  pr[3000 + 8 * l + 7], (pr[3 * l + 2] - pr[3 * l + 1]) * 1e-3);
        const int nl = std::min(hc.nlevels, 999);
        double a = 0, b = 0, c = 0;
        for (int l = 0; l + 1 < nl; ++l) {
          a += pr[3 * l + 1] - pr[3 * l];
          b += pr[3 * l + 2] - pr[3 * l + 1];
          c += pr[3 * l + 3] - pr[3 * l + 2];
        }
        fprintf(stderr, "k_levels: %d levels, grid %d x %d: phase A %.1f us, phase B %.1f us, "
                "between %.1f us\n", hc.nlevels, nsm, per_sm, a * 1e-3, b * 1e-3, c * 1e-3);
      }
      if (!hc.abort) {
        P.root_vol = hc.root_vol;
        total = hc.total;
        if (total == 0) return 0;  // empty tree
        std::vector<long long> lb(hc.nlevels + 1);
        VS_TRY(d2h(lb.data(), lv_lb.p, lb.size() * sizeof(long long), st));
        level_base.assign(lb.begin(), lb.end());
      }
    }
  }
  if (total < 0) {
  level_base.clear();
  VS_TRY(arrays(1));
  VS_TRY(cur.ensure(sizeof(Box), "level"));
  {
    // root_vol is needed by every level's halting rule: read the bbox with the header
    k_root_level<<<1, 32, 0, st>>>(dbb, cur.as<Box>(), prep_ctx(), dh);
    VS_TRY(check_launch("k_root_level"));
    VS_TRY(scan_level(dh, 1));
    int rb[6];
    VS_CUDA(cudaMemcpyAsync(rb, dbb, sizeof rb, cudaMemcpyDeviceToHost, st), "bbox d2h");
    VS_TRY(d2h(hh, dh, sizeof hh, st));
    if (rb[3] < 0) return 0;  // empty tree
    P.root_vol = (int64_t)(rb[3] - rb[0]) * (rb[4] - rb[1]) * (rb[5] - rb[2]);
  }

  int64_t n = hh[0], base = 0;
  int level = 0;
  while (n > 0) {
    level_base.push_back(base);
    KdLevel L;
    L.n = (int)n;
    L.box = cur.as<Box>();
    for (int k = 0; k < KA; ++k) L.off[k] = arr(k);
    const int64_t* tot = hh + 1;
    VS_TRY(dec.ensure(n * sizeof(KdDecision), "decisions"));
    VS_TRY(cnt.ensure((n + 1) * sizeof(int64_t), "counts"));
    BinnedCtx B;
    B.nc[0] = ncx; B.nc[1] = ncy; B.nc[2] = ncz;
    if (!binned) {
      VS_TRY(spx.ensure((tot[A_X] + 1) * sizeof(Span), "span_x"));
      VS_TRY(spy.ensure((tot[A_Y] + 1) * sizeof(Span), "span_y"));
      VS_TRY(spz.ensure((tot[A_Z] + 32) * sizeof(Span), "span_z"));
      VS_TRY(pxz.ensure((tot[A_PXZ] + 1) * 4, "pxz"));
      VS_TRY(pyz.ensure((tot[A_PYZ] + 1) * 4, "pyz"));
      VS_TRY(scr.ensure((tot[A_SCR] + 1) * sizeof(RBox), "scratch"));
      if (tot[A_X] > 0) {
        // some pass merges chunks with atomics: any x/y-chunked node (> 64 rows) is also
        // z-chunked (> 32 projection rows), and per node A_IZ >= A_ZW with equality iff not
        if (tot[A_IZ] > tot[A_ZW]) {
          const int64_t mx = std::max(std::max(std::max(tot[A_X], tot[A_Y]), tot[A_Z]),
                                      std::max(tot[A_PXZ], tot[A_PYZ]));
          k_span_init<<<grid_for(mx, 256), 256, 0, st>>>(
              spx.as<Span>(), tot[A_X], spy.as<Span>(), tot[A_Y], spz.as<Span>(), tot[A_Z],
              pxz.as<uint32_t>(), tot[A_PXZ], pyz.as<uint32_t>(), tot[A_PYZ]);
          VS_TRY(check_launch("k_span_init"));
        }
        // the x and y passes are independent: the y pass runs on a side stream concurrently
        VS_CUDA(cudaEventRecord(ev_fork, st), "fork");
        VS_CUDA(cudaStreamWaitEvent(side, ev_fork, 0), "fork wait");
        k_spans_rows<1><<<grid_for(tot[A_IY], 8), 256, 0, side>>>(bits, ny, nzw, L, tot[A_IY],
                                                                  spy.as<Span>(),
                                                                  pyz.as<uint32_t>());
        VS_TRY(check_launch("k_spans_rows<y>"));
        VS_CUDA(cudaEventRecord(ev_join, side), "join");
        k_spans_rows<0><<<grid_for(tot[A_IX], 8), 256, 0, st>>>(bits, ny, nzw, L, tot[A_IX],
                                                                spx.as<Span>(), pxz.as<uint32_t>());
        VS_TRY(check_launch("k_spans_rows<x>"));
        VS_CUDA(cudaStreamWaitEvent(st, ev_join, 0), "join wait");
        k_spans_z<<<grid_for(tot[A_IZ], 8), 256, 0, st>>>(L, tot[A_IZ], pxz.as<uint32_t>(),
                                                          pyz.as<uint32_t>(), spz.as<Span>());
        VS_TRY(check_launch("k_spans_z"));
      }
      // top levels (few, big nodes): spans staged in shared memory; wide levels: more blocks
      if (n <= 512)
        k_decide<true><<<(unsigned)n, DT, 0, st>>>(L, P, spx.as<Span>(), spy.as<Span>(),
                                                   spz.as<Span>(), scr.as<RBox>(), B,
                                                   dec.as<KdDecision>(), cnt.as<int64_t>());
      else
        k_decide<false><<<(unsigned)n, DT, 0, st>>>(L, P, spx.as<Span>(), spy.as<Span>(),
                                                    spz.as<Span>(), scr.as<RBox>(), B,
                                                    dec.as<KdDecision>(), cnt.as<int64_t>());
      VS_TRY(check_launch("k_decide"));
    } else {
      if (level == 0) {
        const int64_t ncell = (int64_t)ncx * ncy * ncz;
        VS_TRY(cellb.ensure(ncell * sizeof(CBox), "cells"));
        VS_TRY(launch_cell_boxes(bits, nx, ny, nz, cs, ncx, ncy, ncz, cellb.as<CBox>(), st));
        if (cs <= CPK_MAX_CS) {  // packed copies for the cell-slab passes
          VS_TRY(cpk.ensure(2 * ncell * sizeof(uint32_t), "packed cells"));
          k_cell_pack<<<(unsigned)cdiv(ncell, 256), 256, 0, st>>>(
              cellb.as<CBox>(), ncx, ncy, ncz, cs, cpk.as<uint32_t>(), cpk.as<uint32_t>() + ncell);
          VS_TRY(check_launch("k_cell_pack"));
        }
      }
      const int64_t ncell_all = (int64_t)ncx * ncy * ncz;
      B.cells = cellb.as<CBox>();
      const int64_t t0 = tot[A_C0], t1 = tot[A_C1], t2 = tot[A_C2];
      VS_TRY(cslab.ensure((t0 + t1 + t2 + 3) * sizeof(CBox), "cell slabs"));
      CBox* cbase = cslab.as<CBox>();
      CBox* cs3[3] = {cbase, cbase + t0 + 1, cbase + t0 + t1 + 2};
      if (tot[A_IC0] > t0 || tot[A_IC1] > t1 || tot[A_IC2] > t2) {  // some slab is chunked
        k_cbox_init<<<grid_for(t0 + t1 + t2 + 3, 256), 256, 0, st>>>(cbase, t0 + t1 + t2 + 3);
        VS_TRY(check_launch("k_cbox_init"));
      }
      for (int a = 0; a < 3; ++a) {
        B.cslab[a] = cs3[a];
        B.coff[a] = L.off[A_C0 + a];
      }
      if (cs <= CPK_MAX_CS) {  // packed cells: the three axes in one launch
        const int64_t mi = std::max(std::max(tot[A_IC0], tot[A_IC1]), tot[A_IC2]);
        if (mi > 0) {
          const uint32_t* p0 = cpk.as<uint32_t>();
          k_cell_slabs_pk3<<<dim3(grid_for(mi, 8), 3), 256, 0, st>>>(
              p0, p0 + ncell_all, ncx, ncy, ncz, cs, L, tot[A_IC0], tot[A_IC1], tot[A_IC2],
              cs3[0], cs3[1], cs3[2]);
          VS_TRY(check_launch("k_cell_slabs_pk3"));
        }
      } else {
        // the three axes' cell-slab passes are independent: y and z on the side stream
        VS_CUDA(cudaEventRecord(ev_fork, st), "fork");
        VS_CUDA(cudaStreamWaitEvent(side, ev_fork, 0), "fork wait");
        for (int a = 0; a < 3; ++a) {
          const int64_t items = tot[A_IC0 + a];
          if (items > 0)
            k_cell_slabs<<<grid_for(items, 8), 256, 0, a == 0 ? st : side>>>(
                cellb.as<CBox>(), ncx, ncy, ncz, cs, a, L, items, cs3[a]);
          VS_TRY(check_launch("k_cell_slabs"));
        }
        VS_CUDA(cudaEventRecord(ev_join, side), "join");
        VS_CUDA(cudaStreamWaitEvent(st, ev_join, 0), "join wait");
      }
      if (n <= BINNED_NARROW)  // a few big nodes: one CTA of 8 warps per node
        (cs == 8 ? k_decide_binned<8, VS_BINNED_WPN> : k_decide_binned<0, VS_BINNED_WPN>)
            <<<(unsigned)n, 32 * VS_BINNED_WPN, 0, st>>>(
            L, P, B, dec.as<KdDecision>(), cnt.as<int64_t>());
      else
        (cs == 8 ? k_decide_binned<8, 1> : k_decide_binned<0, 1>)<<<(unsigned)cdiv(n, 4), 128, 0,
                                                                   st>>>(
            L, P, B, dec.as<KdDecision>(), cnt.as<int64_t>());
      VS_TRY(check_launch("k_decide"));
      // exact shrink for the binned leaves (kdtree.py:474)
      if (VS_SHRINK_WARP && P.mls >= 0 && P.mls <= 64)  // leaf extents <= mls
        k_leaf_shrink_warp<<<(unsigned)std::min<int64_t>(cdiv(n, 4), 148 * 16), 128, 0, st>>>(
            bits, ny, nzw, L, dec.as<KdDecision>());
      else
        k_leaf_shrink<<<(unsigned)std::min<int64_t>(n, 148 * 16), 128, 0, st>>>(
            bits, ny, nzw, L, dec.as<KdDecision>());
      VS_TRY(check_launch("k_leaf_shrink"));
    }
    // next level: child offsets, rows of this level, next boxes and their work sizes
    {
      ScanSet S;
      S.k = 1;
      S.a[0] = cnt.as<int64_t>();
      S.totals[0] = dh + KA + 1;
      VS_TRY(scan_arrays(S, nullptr, n, n));
      VS_TRY(check_launch("k_multi_scan"));
    }
    if ((size_t)(base + n) * sizeof(NodeRec) > rec.cap) {  // grow the records (copy-preserving)
      DBuf bigger;
      bigger.st = st;
      VS_TRY(bigger.ensure(std::max<size_t>((base + n) * sizeof(NodeRec) * 2, 4096), "records"));
      if (base) VS_CUDA(cudaMemcpyAsync(bigger.p, rec.p, base * sizeof(NodeRec),
                                        cudaMemcpyDeviceToDevice, st), "records copy");
      std::swap(rec.p, bigger.p);
      std::swap(rec.cap, bigger.cap);
    }
    VS_TRY(nxt.ensure(2 * n * sizeof(Box), "next level"));
    VS_TRY(arrays(2 * n));  // this level's arrays are dead from here on
    k_emit_level<<<(unsigned)cdiv(n, 128), 128, 0, st>>>(dec.as<KdDecision>(), cnt.as<int64_t>(),
                                                         (int)n, base, base + n, level,
                                                         rec.as<NodeRec>(), nxt.as<Box>(),
                                                         prep_ctx());
    VS_TRY(check_launch("k_emit_level"));
    VS_TRY(scan_level(dh + KA + 1, 2 * n));
    VS_TRY(d2h(hh, dh, sizeof hh, st));  // the next level's totals and (KA + 1) its node count
    std::swap(cur.p, nxt.p);
    std::swap(cur.cap, nxt.cap);
    base += n;
    n = hh[KA + 1];
    ++level;
  }
  total = base;
  level_base.push_back(total);
  }  // level-by-level path
  // deferred nodes: one CTA per subtree
  DBuf subl, subc, subh, subo, pool, chunks;
  for (DBuf* b : {&subl, &subc, &subh, &subo, &pool, &chunks}) b->st = st;
  SubCtx SC = {};
  int64_t nsub = 0;
  if (P.subtrees && total > 0) {
    VS_TRY(subl.ensure(total * sizeof(int), "subtree list"));
    VS_CUDA(cudaMemsetAsync(dh, 0, 2 * sizeof(int64_t), st), "subtree count");
    k_collect_sub<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(rec.as<NodeRec>(), total,
                                                            subl.as<int>(), dh, dh + 1);
    VS_TRY(check_launch("k_collect_sub"));
    int64_t cnt2[2];
    VS_TRY(d2h(cnt2, dh, sizeof cnt2, st));
    nsub = cnt2[0];
    if (nsub > 0) {
      VS_TRY(subc.ensure(nsub * sizeof(int), "subtree counts"));
      VS_TRY(subh.ensure(nsub * sizeof(int), "subtree heights"));
      VS_TRY(subo.ensure(nsub * sizeof(int), "subtree chunk offsets"));
      const size_t smem = ((sizeof(SubSmem) + 15) & ~size_t(15)) + SUB_WORDS * sizeof(uint32_t);
      VS_CUDA(cudaFuncSetAttribute(k_subtrees, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem), "k_subtrees smem");
      int64_t pool_chunks = std::max<int64_t>(cnt2[1], 1024);  // k_collect_sub's estimate
      const int* order = nullptr;
      DBuf sord;
      sord.st = st;
      if (VS_SUB_LPT && nsub > 1) {  // biggest subtrees first
        VS_TRY(sord.ensure((2 * SUB_CLASSES + nsub) * sizeof(int), "subtree order"));
        int* hist = sord.as<int>();
        VS_CUDA(cudaMemsetAsync(hist, 0, 2 * SUB_CLASSES * sizeof(int), st), "subtree classes");
        const unsigned g = (unsigned)cdiv(nsub, 256);
        k_sub_class<<<g, 256, 0, st>>>(rec.as<NodeRec>(), subl.as<int>(), nsub, hist);
        VS_TRY(check_launch("k_sub_class"));
        k_sub_order<<<g, 256, 0, st>>>(rec.as<NodeRec>(), subl.as<int>(), nsub, hist,
                                       hist + SUB_CLASSES, hist + 2 * SUB_CLASSES);
        VS_TRY(check_launch("k_sub_order"));
        order = hist + 2 * SUB_CLASSES;
      }
      for (;;) {
        VS_TRY(pool.ensure(pool_chunks * SUB_CHUNK * sizeof(SubRow), "subtree rows"));
        VS_TRY(chunks.ensure((pool_chunks + nsub) * sizeof(int), "subtree chunks"));
        VS_CUDA(cudaMemsetAsync(dh + 1, 0, 3 * sizeof(int64_t), st), "subtree counters");
        SC.rec = rec.as<NodeRec>();
        SC.list = subl.as<int>();
        SC.pool = pool.as<SubRow>();
        SC.pool_chunks = pool_chunks;
        SC.pool_used = reinterpret_cast<unsigned long long*>(dh + 1);
        SC.chunks_used = reinterpret_cast<unsigned long long*>(dh + 2);
        SC.status = reinterpret_cast<int*>(dh + 3);
        SC.count = subc.as<int>();
        SC.height = subh.as<int>();
        SC.choff = subo.as<int>();
        SC.chunks = chunks.as<int>();
        SC.order = order;
        k_subtrees<<<(unsigned)nsub, SUB_T, smem, st>>>(bits, ny, nzw, P, SC);
        VS_TRY(check_launch("k_subtrees"));
        int64_t res[3];
        VS_TRY(d2h(res, dh + 1, sizeof res, st));
        const char* penv2 = getenv("VSB200_KD_PROFILE");
        if (penv2 && penv2[0] == '1') {  // dev profile: the subtrees' row counts
          std::vector<int> cnts(nsub);
          VS_TRY(d2h(cnts.data(), subc.p, nsub * sizeof(int), st));
          long long sum = 0;
          int mx = 0;
          for (int c : cnts) { sum += c; mx = std::max(mx, c); }
          fprintf(stderr, "k_subtrees: %lld subtrees, %lld rows, largest %d rows\n",
                  (long long)nsub, sum, mx);
        }
        const int status = (int)(res[2] & 0xffffffff);
        if (status & 2) return KD_RETRY_LEVELS;
        if (!(status & 1)) break;
        pool_chunks = std::max<int64_t>(2 * pool_chunks, res[0] + res[0] / 4);
      }
    }
  }
  VS_TRY(sizes.ensure(total * sizeof(int), "sizes"));
  VS_TRY(pre.ensure(total * sizeof(int), "preorder"));
  const int nlev = (int)level_base.size() - 1;
  int order_grid = 0;  // co-resident blocks for k_order_levels_grid (0: not used)
  if (VS_ORDER_GRID && total > VS_ORDER_GRID_MIN) {
    int per_sm = 0, nsm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_order_levels_grid, 1024, 0) ==
            cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      order_grid = per_sm * nsm;
    cudaGetLastError();
  }
  if (total <= (1 << 16) || order_grid > 0) {
    DBuf lb;
    lb.st = st;
    VS_TRY(lb.ensure(level_base.size() * sizeof(int64_t), "level bases"));
    VS_CUDA(cudaMemcpyAsync(lb.p, level_base.data(), level_base.size() * sizeof(int64_t),
                            cudaMemcpyHostToDevice, st), "level bases");
    if (order_grid > 0) {
      const NodeRec* rp = rec.as<NodeRec>();
      const int64_t* lbp = lb.as<int64_t>();
      const int* scp = subc.as<int>();
      int* szp = sizes.as<int>();
      int* prp = pre.as<int>();
      void* args[] = {&rp, &lbp, (void*)&nlev, &scp, &szp, &prp};
      VS_CUDA(cudaLaunchCooperativeKernel((void*)k_order_levels_grid, dim3(order_grid),
                                          dim3(1024), args, 0, st), "k_order_levels_grid");
    } else {
      k_order_levels<<<1, 1024, 0, st>>>(rec.as<NodeRec>(), lb.as<int64_t>(), nlev,
                                         subc.as<int>(), sizes.as<int>(), pre.as<int>());
      VS_TRY(check_launch("k_order_levels"));
    }
  } else {
    for (int l = nlev - 1; l >= 0; --l) {
      const int64_t b0 = level_base[l], b1 = level_base[l + 1];
      k_sizes<<<(unsigned)cdiv(b1 - b0, 128), 128, 0, st>>>(rec.as<NodeRec>(), b0, b1,
                                                            subc.as<int>(), sizes.as<int>());
      VS_TRY(check_launch("k_sizes"));
    }
    VS_CUDA(cudaMemsetAsync(pre.p, 0, sizeof(int), st), "pre root");
    for (int l = 0; l < nlev; ++l) {
      const int64_t b0 = level_base[l], b1 = level_base[l + 1];
      k_preorder<<<(unsigned)cdiv(b1 - b0, 128), 128, 0, st>>>(rec.as<NodeRec>(), b0, b1,
                                                               sizes.as<int>(), pre.as<int>());
      VS_TRY(check_launch("k_preorder"));
    }
  }
  int m = 0;
  VS_TRY(d2h(&m, sizes.p, sizeof m, st));
  R->m = m;
  if (m == 0) return 0;
  VS_TRY(R->lo.ensure(3 * m * 4, "lo"));
  VS_TRY(R->hi.ensure(3 * m * 4, "hi"));
  VS_TRY(R->axis.ensure(m, "axis"));
  VS_TRY(R->plane.ensure(m * 4, "plane"));
  VS_TRY(R->left.ensure(m * 4, "left"));
  VS_TRY(R->right.ensure(m * 4, "right"));
  VS_CUDA(cudaMemsetAsync(dbb, 0, sizeof(int), st), "height init");
  k_scatter_rows<<<(unsigned)cdiv(total, 128), 128, 0, st>>>(
      rec.as<NodeRec>(), total, sizes.as<int>(), pre.as<int>(), R->lo.as<int32_t>(),
      R->hi.as<int32_t>(), R->axis.as<int8_t>(), R->plane.as<int32_t>(), R->left.as<int32_t>(),
      R->right.as<int32_t>(), dbb);
  VS_TRY(check_launch("k_scatter_rows"));
  if (nsub > 0) {
    k_scatter_sub<<<(unsigned)nsub, 128, 0, st>>>(
        rec.as<NodeRec>(), subl.as<int>(), SC, pre.as<int>(), R->lo.as<int32_t>(),
        R->hi.as<int32_t>(), R->axis.as<int8_t>(), R->plane.as<int32_t>(), R->left.as<int32_t>(),
        R->right.as<int32_t>(), dbb);
    VS_TRY(check_launch("k_scatter_sub"));
  }
  VS_TRY(d2h(&R->height, dbb, sizeof(int), st));
  R->root = 0;
  return 0;
}

}  // namespace

extern "C" {

int vs_kd_build(const uint32_t* bits, int nx, int ny, int nz, int deep, int mls, int binned,
                int bins, int cs, void** handle, vs_stream_t stream) {
  return vs_kd_build_bbox(bits, nx, ny, nz, nullptr, deep, mls, binned, bins, cs, handle, stream);
}

int vs_kd_build_bbox(const uint32_t* bits, int nx, int ny, int nz, const int* bbox, int deep,
                     int mls, int binned, int bins, int cs, void** handle, vs_stream_t stream) {
  if (!bits || !handle || nx < 1 || ny < 1 || nz < 1 || bins < 2 || cs < 1)
    return fail_arg("vs_kd_build");
  if (bins > 65) return fail_arg("vs_kd_build: bins > 65");
  if (nz > 1024) return fail_arg("vs_kd_build: nz > 1024");
  cudaStream_t st = S(stream);
  auto* R = new KdResultImpl();
  *handle = R;
  for (DBuf* b : {&R->lo, &R->hi, &R->axis, &R->plane, &R->left, &R->right}) b->st = st;
  // VSB200_KD_SUBTREES=0: every level through the level loop (A/B and tests)
  const char* env = getenv("VSB200_KD_SUBTREES");
  const int subtrees = !(env && env[0] == '0');
  // VSB200_KD_DEVLEVELS=0: the big-node levels through the host loop instead of k_levels
  const char* env2 = getenv("VSB200_KD_DEVLEVELS");
  const int dev_levels = !(env2 && env2[0] == '0');
  int rc = kd_build(bits, nx, ny, nz, deep, mls, binned, bins, cs, bbox, subtrees, dev_levels, R,
                    st);
  if (rc == KD_RETRY_LEVELS)
    rc = kd_build(bits, nx, ny, nz, deep, mls, binned, bins, cs, bbox, 0, 0, R, st);
  return rc;
}

int vs_kd_result_info(void* handle, int64_t* m, int* root, int* height) {
  auto* R = static_cast<KdResultImpl*>(handle);
  if (!R) return fail_arg("vs_kd_result_info");
  if (m) *m = R->m;
  if (root) *root = R->root;
  if (height) *height = R->height;
  return 0;
}

int vs_kd_result_copy(void* handle, int32_t* lo, int32_t* hi, int8_t* axis, int32_t* plane,
                      int32_t* left, int32_t* right, vs_stream_t stream) {
  auto* R = static_cast<KdResultImpl*>(handle);
  if (!R) return fail_arg("vs_kd_result_copy");
  if (R->m == 0) return 0;
  cudaStream_t st = S(stream);
  const int64_t m = R->m;
  VS_CUDA(cudaMemcpyAsync(lo, R->lo.p, 12 * m, cudaMemcpyDeviceToDevice, st), "copy lo");
  VS_CUDA(cudaMemcpyAsync(hi, R->hi.p, 12 * m, cudaMemcpyDeviceToDevice, st), "copy hi");
  VS_CUDA(cudaMemcpyAsync(axis, R->axis.p, m, cudaMemcpyDeviceToDevice, st), "copy axis");
  VS_CUDA(cudaMemcpyAsync(plane, R->plane.p, 4 * m, cudaMemcpyDeviceToDevice, st), "copy plane");
  VS_CUDA(cudaMemcpyAsync(left, R->left.p, 4 * m, cudaMemcpyDeviceToDevice, st), "copy left");
  VS_CUDA(cudaMemcpyAsync(right, R->right.p, 4 * m, cudaMemcpyDeviceToDevice, st), "copy right");
  return 0;
}

void vs_kd_result_free(void* handle) { delete static_cast<KdResultImpl*>(handle); }

}  // extern "C"

// ---- single-box plane searches (sweep_best_plane kdtree.py:244-262, binned_best_plane
//      kdtree.py:371-381): the level machinery on a one-node level ----------------------------
namespace vs {

__global__ void __launch_bounds__(DT) k_best_plane(KdLevel L, KdParams P,
                                                   const Span* __restrict__ span_x,
                                                   const Span* __restrict__ span_y,
                                                   const Span* __restrict__ span_z,
                                                   RBox* __restrict__ scratch, BinnedCtx B,
                                                   long long* __restrict__ out) {
  __shared__ DecideSmem sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Box b = L.box[0];
  const int ext[3] = {b.hi[0] - b.lo[0], b.hi[1] - b.lo[1], b.hi[2] - b.lo[2]};
  long long found = 0, axis = -1, pos = 0, cost = 0;
  if (!P.binned) {
    const Span* sp[3] = {span_x, span_y, span_z};
    const RBox t = range_box(span_x, 0, ext[0], sm);
    if (t.hi0 >= 0) {
      const int64_t tv = rvol(t);  // _region_tight_volume
      int ba = -1, bk = 0;
      int64_t bc = 0;
      for (int a = 0; a < 3; ++a) {
        if (ext[a] < 2) continue;
        int k;
        int64_t c;
        sweep_axis(sp[a], ext[a], scratch, sm, k, c);
        if (ba >= 0 && c >= bc) continue;
        ba = a; bk = k; bc = c;
      }
      if (ba >= 0 && bc < tv) { found = 1; axis = ba; pos = b.lo[ba] + bk; cost = bc; }
    }
  } else if (warp == 0) {
    Box target;
    if (cells_reduce(B, 0, b, 0, b, P.cs, lane, target)) {
      int ba = -1, bp = 0;
      int64_t bc = 0;
      for (int a = 0; a < 3; ++a) {
        int ps[64];
        const int np = snapped_positions(b.lo[a], b.hi[a], P.bins, P.cs, ps);
        for (int q = 0; q < np; ++q) {
          Box lreg = b, rreg = b, lb, rb;
          lreg.hi[a] = ps[q];
          rreg.lo[a] = ps[q];
          const bool l = cells_reduce(B, 0, b, a, lreg, P.cs, lane, lb);
          const bool r = cells_reduce(B, 0, b, a, rreg, P.cs, lane, rb);
          const int64_t c = (l ? box_vol(lb) : 0) + (r ? box_vol(rb) : 0);
          if (ba < 0 || c < bc) { ba = a; bp = ps[q]; bc = c; }
        }
      }
      if (ba >= 0 && bc < box_vol(target)) { found = 1; axis = ba; pos = bp; cost = bc; }
    }
  }
  if (threadIdx.x == 0) { out[0] = found; out[1] = axis; out[2] = pos; out[3] = cost; }
}

// precompute_cell_boxes layout (kdtree.py:285-320): C-order lo/hi with the reference's
// placeholders for empty cells (lo = c*cs, hi = (c+1)*cs, unclipped).
__global__ void k_cell_box_rows(const CBox* __restrict__ cells, int ncx, int ncy, int ncz, int cs,
                                int32_t* __restrict__ lo, int32_t* __restrict__ hi,
                                uint8_t* __restrict__ occ) {
  const int64_t n = (int64_t)ncx * ncy * ncz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cz = (int)(i % ncz), cy = (int)((i / ncz) % ncy), cx = (int)(i / ((int64_t)ncz * ncy));
  const int c[3] = {cx, cy, cz};
  const CBox v = cells[i];
  const bool o = v.lo[0] != KD_FAR;
  occ[i] = o;
  for (int k = 0; k < 3; ++k) {
    lo[3 * i + k] = o ? v.lo[k] : c[k] * cs;
    hi[3 * i + k] = o ? v.hi[k] : (c[k] + 1) * cs;
  }
}

}  // namespace vs

extern "C" {

int vs_cell_boxes(const uint32_t* bits, int nx, int ny, int nz, int cs, int32_t* lo, int32_t* hi,
                  uint8_t* occupied, vs_stream_t stream) {
  if (!bits || !lo || !hi || !occupied || nx < 1 || ny < 1 || nz < 1 || cs < 1)
    return fail_arg("vs_cell_boxes");
  cudaStream_t st = S(stream);
  const int ncx = (int)cdiv(nx, cs), ncy = (int)cdiv(ny, cs), ncz = (int)cdiv(nz, cs);
  const int64_t n = (int64_t)ncx * ncy * ncz;
  DBuf cells;
  cells.st = st;
  VS_TRY(cells.ensure(n * sizeof(CBox), "cells"));
  VS_TRY(launch_cell_boxes(bits, nx, ny, nz, cs, ncx, ncy, ncz, cells.as<CBox>(), st));
  k_cell_box_rows<<<(unsigned)cdiv(n, 128), 128, 0, st>>>(cells.as<CBox>(), ncx, ncy, ncz, cs, lo,
                                                          hi, occupied);
  VS_TRY(check_launch("k_cell_box_rows"));
  VS_CUDA(cudaStreamSynchronize(st), "sync");
  return 0;
}

int vs_kd_best_plane(const uint32_t* bits, int nx, int ny, int nz, const int* box_host,
                     int binned, int bins, int cs, long long* out_host, vs_stream_t stream) {
  if (!bits || !box_host || !out_host || nx < 1 || ny < 1 || nz < 1 || bins < 2 || bins > 65 ||
      cs < 1)
    return fail_arg("vs_kd_best_plane");
  if (nz > 1024) return fail_arg("vs_kd_best_plane: nz > 1024");
  cudaStream_t st = S(stream);
  out_host[0] = 0; out_host[1] = -1; out_host[2] = 0; out_host[3] = 0;
  Box b;
  const int dims[3] = {nx, ny, nz};
  for (int k = 0; k < 3; ++k) { b.lo[k] = box_host[k]; b.hi[k] = box_host[3 + k]; }
  if (!binned) {  // sweep_best_plane clips the box to the volume first
    for (int k = 0; k < 3; ++k) {
      b.lo[k] = std::max(b.lo[k], 0);
      b.hi[k] = std::min(b.hi[k], dims[k]);
      if (b.lo[k] >= b.hi[k]) return 0;
    }
  }
  const int ext[3] = {b.hi[0] - b.lo[0], b.hi[1] - b.lo[1], b.hi[2] - b.lo[2]};
  for (int k = 0; k < 3; ++k)
    if (ext[k] <= 0) return 0;
  const int wz = (ext[2] + 31) / 32;
  const int ncx = (int)cdiv(nx, cs), ncy = (int)cdiv(ny, cs), ncz = (int)cdiv(nz, cs);
  const int nc[3] = {ncx, ncy, ncz};
  DBuf lev, spx, spy, spz, pxz, pyz, scr, cellb, cslab, res;
  for (DBuf* d : {&lev, &spx, &spy, &spz, &pxz, &pyz, &scr, &cellb, &cslab, &res}) d->st = st;
  // one-node level: box + KA offset arrays of 2 entries
  struct Host {
    Box box;
    int64_t off[KA][2];
  } h;
  memset(&h, 0, sizeof h);
  h.box = b;
  const int64_t sizes[A_IZ + 1] = {ext[0], ext[1], ext[2], (int64_t)ext[0] * wz,
                                   (int64_t)ext[1] * wz, wz,
                                   std::max(ext[0], std::max(ext[1], ext[2])),
                                   span_items(ext[0], ext[1]),
                                   span_items(ext[1], ext[0]),
                                   (int64_t)wz * cdiv(std::max(ext[0], ext[1]), 32)};
  for (int k = 0; k <= A_IZ; ++k) h.off[k][1] = sizes[k];
  int64_t csz[3], cit[3];
  for (int a = 0; a < 3; ++a) {
    int c0 = std::max(b.lo[a] / cs, 0), c1 = std::min((b.hi[a] - 1) / cs, nc[a] - 1);
    csz[a] = std::max(c1 - c0 + 1, 0);
    h.off[A_C0 + a][1] = csz[a];
  }
  for (int a = 0; a < 3; ++a) {
    const int o1 = a == 0 ? 1 : 0, o2 = a == 2 ? 1 : 2;
    cit[a] = csz[a] * cdiv(csz[o1] * csz[o2], CELL_CHUNK);
    h.off[A_IC0 + a][1] = cit[a];
  }
  VS_TRY(lev.ensure(sizeof h, "level"));
  VS_CUDA(cudaMemcpyAsync(lev.p, &h, sizeof h, cudaMemcpyHostToDevice, st), "level copy");
  Host* d = lev.as<Host>();
  KdLevel L;
  L.n = 1;
  L.box = &d->box;
  for (int k = 0; k < KA; ++k) L.off[k] = d->off[k];
  KdParams P;
  P.deep = 1; P.mls = -1; P.binned = binned; P.bins = bins; P.cs = cs; P.root_vol = 0;
  BinnedCtx B;
  B.nc[0] = ncx; B.nc[1] = ncy; B.nc[2] = ncz;
  const int nzw = (int)nzw_of(nz);
  VS_TRY(res.ensure(4 * sizeof(long long), "result"));
  VS_TRY(scr.ensure((std::max(ext[0], std::max(ext[1], ext[2])) + 1) * sizeof(RBox), "scratch"));
  if (!binned) {
    VS_TRY(spx.ensure((ext[0] + 1) * sizeof(Span), "span_x"));
    VS_TRY(spy.ensure((ext[1] + 1) * sizeof(Span), "span_y"));
    VS_TRY(spz.ensure((ext[2] + 32) * sizeof(Span), "span_z"));
    VS_TRY(pxz.ensure((sizes[A_PXZ] + 1) * 4, "pxz"));
    VS_TRY(pyz.ensure((sizes[A_PYZ] + 1) * 4, "pyz"));
    const int64_t mx = std::max(std::max(std::max(sizes[A_X], sizes[A_Y]), sizes[A_Z]),
                                std::max(sizes[A_PXZ], sizes[A_PYZ]));
    k_span_init<<<grid_for(mx, 256), 256, 0, st>>>(
        spx.as<Span>(), sizes[A_X], spy.as<Span>(), sizes[A_Y], spz.as<Span>(), sizes[A_Z],
        pxz.as<uint32_t>(), sizes[A_PXZ], pyz.as<uint32_t>(), sizes[A_PYZ]);
    k_spans_rows<0><<<grid_for(sizes[A_IX], 8), 256, 0, st>>>(bits, ny, nzw, L, sizes[A_IX],
                                                              spx.as<Span>(), pxz.as<uint32_t>());
    k_spans_rows<1><<<grid_for(sizes[A_IY], 8), 256, 0, st>>>(bits, ny, nzw, L, sizes[A_IY],
                                                              spy.as<Span>(), pyz.as<uint32_t>());
    k_spans_z<<<grid_for(sizes[A_IZ], 8), 256, 0, st>>>(L, sizes[A_IZ], pxz.as<uint32_t>(),
                                                        pyz.as<uint32_t>(), spz.as<Span>());
    VS_TRY(check_launch("spans"));
  } else {
    const int64_t ncell = (int64_t)ncx * ncy * ncz;
    VS_TRY(cellb.ensure(ncell * sizeof(CBox), "cells"));
    VS_TRY(launch_cell_boxes(bits, nx, ny, nz, cs, ncx, ncy, ncz, cellb.as<CBox>(), st));
    B.cells = cellb.as<CBox>();
    VS_TRY(cslab.ensure((csz[0] + csz[1] + csz[2] + 3) * sizeof(CBox), "cell slabs"));
    CBox* cs3[3] = {cslab.as<CBox>(), cslab.as<CBox>() + csz[0] + 1,
                    cslab.as<CBox>() + csz[0] + csz[1] + 2};
    k_cbox_init<<<grid_for(csz[0] + csz[1] + csz[2] + 3, 256), 256, 0, st>>>(
        cslab.as<CBox>(), csz[0] + csz[1] + csz[2] + 3);
    for (int a = 0; a < 3; ++a) {
      k_cell_slabs<<<grid_for(cit[a], 8), 256, 0, st>>>(cellb.as<CBox>(), ncx, ncy, ncz, cs, a, L,
                                                        cit[a], cs3[a]);
      B.cslab[a] = cs3[a];
      B.coff[a] = d->off[A_C0 + a];
    }
    VS_TRY(check_launch("cell slabs"));
  }
  k_best_plane<<<1, DT, 0, st>>>(L, P, spx.as<Span>(), spy.as<Span>(), spz.as<Span>(),
                                 scr.as<RBox>(), B, res.as<long long>());
  VS_TRY(check_launch("k_best_plane"));
  VS_TRY(d2h(out_host, res.p, 4 * sizeof(long long), st));
  return 0;
}

}  // extern "C"
