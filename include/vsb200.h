/*
 * vsb200.h -- C ABI of libvsb200.so, the B200 (sm_100a) implementation of the voxelskip
 * empty-space-skipping hot path (arXiv 1912.09596): TF classification -> hierarchy build
 * (LBVH / macro grid / SVT k-d / binned k-d / hybrid) -> DVR ray march.
 *
 * The reference (`voxelskip`, /root/reference/pkg/src/voxelskip/) is a Python package, so its
 * own "FFI" for this path is the Python call surface listed in SURVEY.md §8(b).  Each entry
 * point below names the reference function it replaces; the Python package
 * paper_1912_09596_b200 binds them through ctypes with the same names and semantics as the
 * reference.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer unless marked (host).  The library never
 *    allocates or frees caller memory; scratch comes from *_workspace() queries (two-phase,
 *    CUB style) and is passed back as (ws, ws_bytes).
 *  - Every call takes an explicit stream (a cudaStream_t) and is asynchronous on it.
 *  - Return value: 0 ok; negative = argument error (VS_E*); positive = a cudaError_t.
 *    vs_last_error() returns the message of the last failure on the calling host thread.
 *  - Volumes are C-order [x][y][z] (z fastest), as volume.py:64-81.  Scalar volumes are held
 *    as uint8 LUT bins (quantize_scalar, volume.py:159-162, is the identity on u8 data).
 *  - Bit volumes are packed along z: word (x, y, w) at (x*ny + y)*ceil(nz/32) + w, bit z&31.
 *  - Boxes are half-open int32 [lo, hi) stored as (rows, 3).
 *  - No floating-point atomics touch any parity output; results are deterministic.
 */
#ifndef VSB200_H
#define VSB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* vs_stream_t; /* cudaStream_t */

enum { VS_OK = 0, VS_EINVAL = -1, VS_ERANGE = -2, VS_EWORKSPACE = -3 };

/* Transfer-function classification parameters (device copy read by the kernels, so a TF
 * change is one 64-byte H2D and CUDA-graph replays stay valid).  Built on the host from the
 * LUT alpha column by vs_tf_params_from_alpha: visible bin <=> lut[bin,3] > 0
 * (classify, volume.py:307-319). */
typedef struct vs_tf_params {
  uint32_t vis[8];   /* 256-bit visibility mask, bit b = (alpha[b] > 0)                   */
  int32_t mode;      /* 0 = table lookup, 1/2 = that many visibility changes, 3 = constant */
  int32_t start;     /* visibility of bin 0                                                */
  int32_t bound[2];  /* bins where visibility flips (ascending), modes 1/2                 */
  int32_t nvisible;  /* number of visible bins                                             */
  int32_t pad[3];
} vs_tf_params;

const char* vs_version(void);
int vs_last_error(char* buf, size_t size);

/* Host helper: alpha (host, 256 floats) -> params (host). */
int vs_tf_params_from_alpha(const float* alpha256, vs_tf_params* out);

/* ---- classification: volume.py:159-162 (quantize_scalar), 289-304 (_dilate26),
 *      307-319 (classify), 322-324 (occupancy) ------------------------------------------ */

/* quantize_scalar: floor(v*255 + 0.5) clipped to [0,255] in float64, f32 field -> u8 bins. */
int vs_quantize_f32(const float* field, int64_t n, uint8_t* bins, vs_stream_t stream);

/* Fused TF pass over the u8 bins, one read of the volume (fast path: nz % 16 == 0, 8^3
 * bricks).  Per 8^3 brick it writes a 27-bit halo summary: bit (ex+1)*9+(ey+1)*3+(ez+1) is
 * set iff the brick holds a visible voxel inside the 1-voxel halo of the neighbour brick at
 * offset -e (e=-1: last slab, 0: anywhere, +1: first slab).  The dilated brick vote of
 * flag_bricks(classify(dilate=True)) (lbvh.py:83-102) is then an OR over 27 neighbours, and
 * bit 13 alone is the undilated vote.  Optionally writes the undilated packed bits; adds the
 * count of visible voxels (occupancy numerator) to *count (caller zeroes it).
 * summary: ceil(nx/8)*ceil(ny/8)*ceil(nz/8) uint32, C-order. */
int vs_classify_summary(const uint8_t* bins, int nx, int ny, int nz, const vs_tf_params* tf,
                        uint32_t* summary, uint32_t* bits_opt, unsigned long long* count_opt,
                        vs_stream_t stream);

/* Generic-dims classification to packed undilated bits (+ optional visible count). */
int vs_classify_bits(const uint8_t* bins, int nx, int ny, int nz, const vs_tf_params* tf,
                     uint32_t* bits, unsigned long long* count_opt, vs_stream_t stream);

/* classify + _dilate26 fused into one pass over the volume (volume.py:307-319 with
 * dilate=True): packed dilated bits + optional visible count of the UNDILATED classification.
 * Needs nz % 32 == 0, nz <= 1024 and a 16-byte aligned volume (VS_EINVAL otherwise). */
int vs_classify_dilate_bits(const uint8_t* bins, int nx, int ny, int nz, const vs_tf_params* tf,
                            uint32_t* bits, unsigned long long* count_opt, vs_stream_t stream);

/* As vs_classify_dilate_bits, plus the tight box of the dilated flags (shrink_to_occupied of
 * the whole volume, the k-d root box, kdtree.py:398) into device int[6] bbox_opt as
 * {lo x, y, z, hi x, y, z} (hi x < 0: no flag), found in the same pass. */
int vs_classify_dilate_bits_bbox(const uint8_t* bins, int nx, int ny, int nz,
                                 const vs_tf_params* tf, uint32_t* bits,
                                 unsigned long long* count_opt, int* bbox_opt,
                                 vs_stream_t stream);

/* _dilate26: 3x3x3 box OR, neighbourhood clipped at the borders.  in != out. */
int vs_dilate_bits(const uint32_t* in, int nx, int ny, int nz, uint32_t* out,
                   vs_stream_t stream);

/* BinaryVolume.bits (bool bytes, C-order) <-> packed bits. */
int vs_pack_bits(const uint8_t* bools, int nx, int ny, int nz, uint32_t* bits,
                 vs_stream_t stream);
int vs_unpack_bits(const uint32_t* bits, int nx, int ny, int nz, uint8_t* bools,
                   vs_stream_t stream);
/* count_nonzero(bits) added to *count (caller zeroes it). */
int vs_count_bits(const uint32_t* bits, int nx, int ny, int nz, unsigned long long* count,
                  vs_stream_t stream);

/* Per-cell vote (any set bit), cells of edge cs clipped at the border, C-order bool bytes:
 * flag_bricks' padded reshape-any (lbvh.py:93-95) and _macro_from_bits (svt.py:161-167). */
int vs_vote_cells(const uint32_t* bits, int nx, int ny, int nz, int cs, uint8_t* flags,
                  vs_stream_t stream);

/* ---- Morton bitmap of non-empty bricks (the sorted order of build_lbvh, lbvh.py:226-229) --
 * A brick grid of nb = (nbx,nby,nbz) bricks is addressed by Morton code in a cube of side
 * P = vs_morton_side(nb) (power of two, >= 8).  Bit `code` of `bitmap` is the brick flag;
 * tile_counts[t] = popcount of the 512-code tile t.  Because Morton codes of distinct bricks
 * are distinct, increasing code order IS the reference's stable argsort of
 * (code << 32 | scan_index). */
int vs_morton_side(int nbx, int nby, int nbz);

/* From the 27-bit summaries (dilate=1 -> flag_bricks(classify(dilate=True)); 0 -> undilated).
 * Also writes the 16^3 macro-cell grid (derive_macro_grid(b, 16), svt.py:134-167) when
 * cell16_opt != NULL: a 16-cell is exactly the OR of its 2x2x2 aligned 8-bricks. */
int vs_summary_to_bitmap(const uint32_t* summary, int nx, int ny, int nz, int dilate, int P,
                         uint32_t* bitmap, uint32_t* tile_counts, uint8_t* cell16_opt,
                         uint32_t* grid_opt, vs_stream_t stream);
/* grid_opt: also the C-order leaf-brick bit grid ((nbx*nby*nbz+31)/32 words) the renderer's
 * brick DDA reads (vs_index_desc.brick_bits), so no separate pass over the brick list. */

/* ---- warm path: TF-independent per-volume brick presence (SURVEY.md §8d "cold / warm") ----
 * presence (vs_presence_words u32): for every 8^3 brick, a 256-bit mask of the u8 bins that
 * occur in the brick's 1-voxel halo (box-clipped).  flag_bricks(classify(v, tf, dilate=True),
 * 8) (lbvh.py:83-102, volume.py:289-319) of any TF is then (presence & visible_bins) != 0 --
 * exact, since the dilated vote of a brick is the OR of base visibility over its halo.  Needs
 * nz % 16 == 0 and 16-byte aligned bins.  vs_presence_to_bitmap: nch channels (<= 4) voting
 * as their union (multichannel semantics); presence_dev_ptrs = device array of the nch
 * channels' presence pointers, tf_params = nch stacked device vs_tf_params blocks. */
int64_t vs_presence_words(int nx, int ny, int nz);
int vs_presence_build(const uint8_t* bins, int nx, int ny, int nz, uint32_t* presence,
                      vs_stream_t stream);
/* The masks of brick x-slabs [bx0, bx1) only (their words: offset bx0 * nby * nbz * 8 of the
 * full array), so N ranks each build a slab range of a replicated volume and one all-gather
 * assembles the array (render.py:16-18's ray-chunk sharding applied to the per-volume pass). */
int vs_presence_build_slab(const uint8_t* bins, int nx, int ny, int nz, int bx0, int bx1,
                           uint32_t* presence, vs_stream_t stream);
int vs_presence_to_bitmap(const uint32_t* const* presence_dev_ptrs, const int32_t* tf_params,
                          int nch, int nx, int ny, int nz, int P, uint32_t* bitmap,
                          uint32_t* tile_counts, uint8_t* cell16_opt, uint32_t* grid_opt,
                          vs_stream_t stream);

/* From C-order brick flag bytes (any brick size). */
int vs_flags_to_bitmap(const uint8_t* flags, int nbx, int nby, int nbz, int P,
                       uint32_t* bitmap, uint32_t* tile_counts, vs_stream_t stream);

/* BrickSet in scan (C) order (flag_bricks, lbvh.py:96-101): coords (n,3), codes (n,).
 * *n_out (device int) receives n. */
size_t vs_bricks_workspace(int nbx, int nby, int nbz);
int vs_bricks_from_bitmap(const uint32_t* bitmap, int nbx, int nby, int nbz, int P,
                          int32_t* coords, uint32_t* codes, int* n_out, void* ws,
                          size_t ws_bytes, vs_stream_t stream);

/* ---- LBVH: build_lbvh (lbvh.py:216-264) = Karras radix tree (lbvh.py:167-200) + refit
 * (lbvh.py:203-213).  Outputs use the reference layout: rows 0..n-2 internal (Karras index),
 * rows n-1..2n-2 the leaves in Morton order; left/right = -1 on leaves; leaf_brick = -1 on
 * internal rows and 0..n-1 on leaves; brick_coords (n,3) Morton-sorted; root 0 (n>0).
 * Capacities: rows >= 2*cap-1, brick_coords >= cap, where cap >= number of bricks.
 * info (device int[2]) receives {n, height} (lbvh.py:128-144).
 * Bitmap path: internal boxes are range reductions over the node's leaf run (no refit climb);
 * info[1] is -1 when n >= 2 (height not computed: vs_lbvh_height fills it on demand, as the
 * reference's Lbvh.height() is computed on call).  brick_grid_opt: the renderer's C-order
 * leaf-brick bit grid ((nbx*nby*nbz+31)/32 words), written in the same launch sequence. */
size_t vs_lbvh_workspace(int P, int64_t cap);
int vs_lbvh_from_bitmap(const uint32_t* bitmap, const uint32_t* tile_counts, int P, int bs,
                        int nx, int ny, int nz, int64_t cap, int32_t* lo, int32_t* hi,
                        int32_t* left, int32_t* right, int32_t* leaf_brick,
                        int32_t* brick_coords, uint32_t* brick_grid_opt, int* info, void* ws,
                        size_t ws_bytes, vs_stream_t stream);
/* Lbvh.height() (lbvh.py:128-144) of a built tree into info[1] (cap = brick capacity). */
size_t vs_lbvh_height_workspace(int64_t cap);
int vs_lbvh_height(const int32_t* left, const int32_t* right, int* info, int64_t cap, void* ws,
                   size_t ws_bytes, vs_stream_t stream);

/* Arbitrary BrickSet (codes may repeat): keys = code << 32 | index, stable radix sort, then
 * the same tree/refit.  n is known to the caller. */
size_t vs_lbvh_bricks_workspace(int64_t n);
int vs_lbvh_from_bricks(const int32_t* coords, const uint32_t* codes, int64_t n, int bs,
                        int nx, int ny, int nz, int32_t* lo, int32_t* hi, int32_t* left,
                        int32_t* right, int32_t* leaf_brick, int32_t* brick_coords, int* info,
                        void* ws, size_t ws_bytes, vs_stream_t stream);


/* ---- renderer: render_frame (render.py:869-911) and the single-ray API (:917-1015) ------ */
enum { VS_KIND_NAIVE = 0, VS_KIND_GRID = 1, VS_KIND_LBVH = 2, VS_KIND_KD = 3, VS_KIND_HYBRID = 4 };
enum { VS_RF_OVERFLOW = 1, VS_RF_ORDER = 2 }; /* render flags */

typedef struct vs_volume_desc {
  const uint8_t* bins;   /* u8 LUT bins, C-order                                      */
  const float* field;    /* float32 field, or NULL when the field is f32(bin/255) exactly */
  int nx, ny, nz, pad;
  /* optional trilinear gather volume (u8 volumes): per voxel the 2x2 (y, z) neighbourhood
   * {(y,z), (y,z+1), (y+1,z), (y+1,z+1)} (+1 clamped) packed in one uint32, so a trilinear
   * sample is two 32-bit loads instead of eight byte loads.  Built by vs_build_quads. */
  const uint32_t* quads;
} vs_volume_desc;

/* Trilinear gather volume for vs_volume_desc.quads: one word per voxel in 4x4x4-voxel tiles
 * (layout internal to the renderer; size vs_quads_words words, < 2^32). */
int64_t vs_quads_words(int nx, int ny, int nz);
int vs_build_quads(const uint8_t* bins, int nx, int ny, int nz, uint32_t* quads,
                   vs_stream_t stream);

/* An index for traversal (render.py:41, index_kind :44-55).
 * grid / hybrid: occ (ncx,ncy,ncz) bool bytes, cell size cs (svt.py:29-37).
 * lbvh: lo/hi (m,3), left/right (m,); root = 0 if lbvh_info[0] (device n_bricks) > 0 else -1
 *       (lbvh_info may be NULL, then `root` is used).
 * kd / hybrid: lo/hi (m,3), axis (m,) int8, plane/left/right (m,), root (kdtree.py:85-127). */
typedef struct vs_index_desc {
  int kind;
  int root;
  const uint8_t* occ;
  int ncx, ncy, ncz, cs;
  const int32_t* lo;
  const int32_t* hi;
  const int32_t* left;
  const int32_t* right;
  const int32_t* plane;
  const int8_t* axis;
  const int* lbvh_info;
  /* lbvh: optional C-order bit grid of the leaf bricks (nbx,nby,nbz) with edge bs; when set,
   * the leaves are enumerated by a brick DDA instead of the tree walk (same intervals). */
  const uint32_t* brick_bits;
  int nbx, nby, nbz, bs;
} vs_index_desc;

/* Orthographic camera with the host-normalised frame of Camera.ray_origins (render.py:134-149):
 * pixel (i, j) starts at (eye + ys*up) + xs*right, xs = ((i + 0.5) - w/2)*scale,
 * ys = ((h/2 - j) - 0.5)*scale, and marches along dir. */
typedef struct vs_camera_desc {
  double eye[3], up[3], right[3], dir[3];
  double scale;
  int width, height;
} vs_camera_desc;

/* Which image rows this launch renders: local row l -> stripe s = l / stripe, image row
 * (s*nparts + part)*stripe + l % stripe (interleaved row stripes for multi-GPU tiles). */
typedef struct vs_rows_desc {
  int nrows, stripe, nparts, part;
} vs_rows_desc;

/* Per-call renderer options (SURVEY §8b threading row: no global mutable state -- every
 * setting travels with the call).  opts == NULL means the defaults below (parity mode). */
enum {
  VS_RO_U8_TABLE = 1,          /* u8 -> f32 through a shared-memory table (same values)     */
  VS_RO_FP64_BINS = 2,         /* every sample's bin in FP64 (no exact FP32 bin filter)      */
  VS_RO_GENERIC_TRAVERSAL = 4, /* generic generator-stack traversal kernel (same intervals)  */
  VS_RO_BRICK_NO_RUNS = 16,    /* brick DDA evaluates every occupied brick's slab            */
  VS_RO_DEFAULT = VS_RO_U8_TABLE
};
typedef struct vs_render_opts {
  /* Early ray termination: a ray stops once its accumulated opacity reaches 1 - ert_eps, so
   * every RGBA channel is within ert_eps of the full integral (LUT colours <= 1) and fewer
   * samples are taken.  <= 0: off, the reference integrator exactly (render.py:758 counts
   * every lattice point; the default). */
  double ert_eps;
  int flags;        /* VS_RO_* code-path bits; all give identical results                */
  int trav_steps;   /* generic kernels: traversal steps per turn (<= 0 unbounded; dflt 1) */
  int sample_steps; /* fused kernel: lattice samples per turn (<= 0 unbounded; dflt 1)    */
  int reserved;
} vs_render_opts;

/* Render rows of a frame.  lut: (256,4) float32 device; corr: 256 float64 device holding
 * 1 - (1 - lut[b,3])^dt computed with libm pow (render.py:752).  Outputs per local row-major
 * pixel: rgba8 (quantised), optional float64 premultiplied rgba, optional per-pixel sample
 * counts; *total_opt += sum of samples (caller zeroes).  *flags |= VS_RF_* on stack overflow
 * or non-monotone interval emission (the host raises).  rows_opt NULL = the full frame. */
int vs_render(const vs_volume_desc* vol, const vs_index_desc* ix, const vs_camera_desc* cam,
              const float* lut, const double* corr, double dt, int nearest,
              const vs_rows_desc* rows_opt, uint8_t* rgba8, double* rgba64_opt,
              int32_t* samples_opt, unsigned long long* total_opt, int* flags, void* ws,
              size_t ws_bytes, int seg_cap, const vs_render_opts* opts, vs_stream_t stream);
/* Two-phase rendering (ws != NULL, seg_cap > 0): a traversal kernel stores each ray's merged
 * segments (up to seg_cap; rays with more are re-traversed inside the integration kernel),
 * then an integration kernel consumes them.  Workspace bytes for npix pixels: */
size_t vs_render_workspace(int64_t npix, int seg_cap);



/* ---- multi-channel volumes (configs[4]; no reference equivalent, see multichannel.cu) ---- */
typedef struct vs_int2 { int32_t x, y; } int2_t;
typedef struct vs_multi_desc {
  int nch, nx, ny, nz;              /* channels (<= 4) and dims                            */
  const uint32_t* quads[4];         /* per channel trilinear gather volume (unused)        */
  const float* lut[4];              /* per channel (256,4) float32 LUT                     */
  const double* corr[4];            /* per channel opacity correction table (libm pow)     */
  const uint32_t* mquads;           /* channel-interleaved gather volume (vs_build_mquads) */
} vs_multi_desc;
/* Channel-interleaved trilinear gather volume: vs_mquads_words(nch) 32-bit words per voxel
 * (1, 2 or 4), word c = channel c's vs_build_quads word, voxels in vs_build_quads' tile order
 * (vs_mquads_size words in all).  bins: nch u8 channel volumes. */
int vs_mquads_words(int nch);
int64_t vs_mquads_size(int nch, int nx, int ny, int nz);
int vs_build_mquads(const uint8_t* const* bins, int nch, int nx, int ny, int nz, uint32_t* out,
                    vs_stream_t stream);
/* dst[i] |= src[i] (OR of per-channel brick summaries). */
int vs_or_words(uint32_t* dst, const uint32_t* src, int64_t n, vs_stream_t stream);
/* Integration of all channels over lattice ranges produced by vs_render_segments. */
int vs_render_multi_integrate(const vs_multi_desc* md, const vs_camera_desc* cam, double dt,
                              const vs_rows_desc* rows_opt, const int2_t* segs, const int* counts,
                              int cap, uint8_t* rgba8, double* rgba64_opt, int32_t* samples_opt,
                              unsigned long long* total_opt, int* flags, vs_stream_t stream);
/* Traversal half of the two-phase renderer alone: per ray lattice ranges (segs: cap x npix
 * int2, ray-minor) and counts (npix). */
int vs_render_segments(const vs_volume_desc* vol, const vs_index_desc* ix,
                       const vs_camera_desc* cam, double dt, const vs_rows_desc* rows_opt,
                       int2_t* segs, int* counts, int cap, int* flags,
                       const vs_render_opts* opts, vs_stream_t stream);

/* Leaf-brick bit grid of an LBVH from its brick_coords (n from n_dev, or cap if NULL). */
int vs_lbvh_brick_grid(const int32_t* brick_coords, const int* n_dev, int64_t cap, int nbx,
                       int nby, int nbz, uint32_t* bits, vs_stream_t stream);

/* traverse_* (render.py:928-961) for a batch of rays: out (nrays, cap, 2) merged intervals,
 * counts[q] = total intervals of ray q (may exceed cap; then out holds the first cap). */
int vs_traverse_rays(const vs_index_desc* ix, int nx, int ny, int nz, const double* origins,
                     const double* dir, int nrays, double* out, int cap, int* counts, int* flags,
                     vs_stream_t stream);

/* integrate (render.py:964-1001) for a batch of rays over given segments. */
int vs_integrate_rays(const vs_volume_desc* vol, const double* origins, const double* dir,
                      const double* segs, const int* counts, int cap, int nrays,
                      const float* lut, const double* corr, double dt, int nearest,
                      double* rgba, long long* samples, vs_stream_t stream);

/* ---- summed-volume tables (svt.py:40-131) ------------------------------------------------ */
/* build_svt_grid: tables (nbx,nby,nbz,bs+1,bs+1,bs+1) uint32, bs in [2, 32]. */
int vs_svt_build(const uint32_t* bits, int nx, int ny, int nz, int bs, uint32_t* tables,
                 vs_stream_t stream);
/* box_count for nbox boxes (lo3, hi3 int32 each, clipped to dims) -> counts (int64). */
int vs_box_count(const uint32_t* tables, int nx, int ny, int nz, int bs, const int32_t* boxes,
                 int nbox, long long* counts, vs_stream_t stream);
/* shrink_to_occupied of one box: out = lo3, hi3 of the set flags inside (hi[0] < 0 = None). */
int vs_tight_box(const uint32_t* bits, int nx, int ny, int nz, const int32_t* box, int* out,
                 vs_stream_t stream);

/* ---- k-d trees: build_kdtree (kdtree.py:387-498) -------------------------------------------
 * Level-synchronous on the device, rows renumbered to the reference's DFS preorder.
 * deep: 0 shallow / 1 deep; mls: max_leaf_size or -1; binned: 0 sweep / 1 binned (bins, cs).
 * Synchronous (one host sync per tree level); scratch is stream-ordered device memory.
 * The result handle is read with vs_kd_result_info / _copy and released with _free. */
int vs_kd_build(const uint32_t* bits, int nx, int ny, int nz, int deep, int mls, int binned,
                int bins, int cs, void** handle, vs_stream_t stream);
/* As vs_kd_build with the root box precomputed on the device (device int[6] from
 * vs_classify_dilate_bits_bbox; NULL: computed from the bits). */
int vs_kd_build_bbox(const uint32_t* bits, int nx, int ny, int nz, const int* bbox, int deep,
                     int mls, int binned, int bins, int cs, void** handle, vs_stream_t stream);
int vs_kd_result_info(void* handle, int64_t* m, int* root, int* height);
int vs_kd_result_copy(void* handle, int32_t* lo, int32_t* hi, int8_t* axis, int32_t* plane,
                      int32_t* left, int32_t* right, vs_stream_t stream);
void vs_kd_result_free(void* handle);

/* precompute_cell_boxes (kdtree.py:285-320) in C order: per cell of edge cs, the tight box of
 * its flags (lo, hi (n,3) int32, global voxel coords; empty cells get the reference's
 * placeholders lo = c*cs, hi = (c+1)*cs) and occupied (n,) bool bytes.  Synchronous. */
int vs_cell_boxes(const uint32_t* bits, int nx, int ny, int nz, int cs, int32_t* lo, int32_t* hi,
                  uint8_t* occupied, vs_stream_t stream);
/* sweep_best_plane (binned = 0; kdtree.py:244-262) or binned_best_plane (binned = 1;
 * kdtree.py:371-381) for one box (host int[6] lo3 hi3).  out (host long long[4]) =
 * {found, axis, position, cost}.  Synchronous. */
int vs_kd_best_plane(const uint32_t* bits, int nx, int ny, int nz, const int* box_host,
                     int binned, int bins, int cs, long long* out_host, vs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VSB200_H */
