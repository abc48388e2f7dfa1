/*
 * vs_oracle.c -- CPU restatement of the voxelskip hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity oracle for the B200 build.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it; the product path
 * (paper_1912_09596_b200/) never links, imports or executes anything under oracle/.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/voxelskip/) with the same arithmetic: IEEE double, no FMA
 * contraction (compiled with -ffp-contract=off), libm pow for the opacity correction,
 * exactly like the numba kernels it mirrors.  The restatement is pinned against golden
 * vectors produced by running the unmodified reference in the build container
 * (tests/golden/make_golden.py); see tests/test_oracle_golden.py.
 *
 * Conventions: volumes and flag volumes are C-order [x][y][z] (z fastest), flags are one
 * byte (0/1) per voxel, boxes are half-open int [lo, hi).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>

typedef int64_t i64;

#define IDX3(x, y, z, ny, nz) ((((i64)(x)) * (ny) + (y)) * (nz) + (z))

static i64 imin64(i64 a, i64 b) { return a < b ? a : b; }
static i64 imax64(i64 a, i64 b) { return a > b ? a : b; }
static i64 floordiv(i64 a, i64 b) { i64 q = a / b; if ((a % b != 0) && ((a < 0) != (b < 0))) q--; return q; }

/* Host threads for the data-parallel loops below (classification, dilation, brick votes).
 * The split is over independent x slabs, so results never depend on the thread count. */
#include <unistd.h>
static int g_threads = 0;
void or_set_threads(int n) { g_threads = n; }
static int nthreads_for(i64 work) {
    int t = g_threads > 0 ? g_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 64) t = 64;
    if ((i64)t > work) t = (int)(work > 0 ? work : 1);
    return t;
}
typedef void (*range_fn)(void* ctx, i64 lo, i64 hi, int tid);
typedef struct { range_fn fn; void* ctx; i64 n; int nt, tid; } ParJob;
static void* par_worker(void* a) {
    ParJob* j = (ParJob*)a;
    i64 lo = j->n * j->tid / j->nt, hi = j->n * (j->tid + 1) / j->nt;
    j->fn(j->ctx, lo, hi, j->tid);
    return NULL;
}
/* fn(ctx, lo, hi, tid) over contiguous chunks of [0, n); returns the thread count used. */
static int par_for(i64 n, range_fn fn, void* ctx) {
    int nt = nthreads_for(n);
    ParJob jobs[64];
    pthread_t th[64];
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].n = n; jobs[t].nt = nt; jobs[t].tid = t;
    }
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, par_worker, &jobs[t]);
    par_worker(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
    return nt;
}

/* ------------------------------------------------------------------------------------ */
/* classification: volume.py:231-234 (quantize_scalar), 361-376 (_dilate26),            */
/* 379-391 (classify), 394-396 (occupancy)                                               */
/* ------------------------------------------------------------------------------------ */

/* volume.py:231-234: floor(v*255 + 0.5) in float64, clipped to [0, 255]. */
static int quantize_f32(float v) {
    double d = floor((double)v * 255.0 + 0.5);
    if (d < 0.0) return 0;
    if (d > 255.0) return 255;
    return (int)d;
}

/* u8 volumes are held by the reference as f32(u/255) (load_raw volume.py:265). */
void or_u8_field_table(float* out256) {
    for (int u = 0; u < 256; ++u) out256[u] = (float)((double)u / 255.0);
}

static float field_value(const void* vol, int is_f32, i64 idx, const float* u8tab) {
    if (is_f32) return ((const float*)vol)[idx];
    return u8tab[((const uint8_t*)vol)[idx]];
}

/* volume.py:361-376: separable 3-tap OR per axis, borders clipped. */
typedef struct { uint8_t* bits; const uint8_t* tmp; i64 nx, ny, nz; int axis; } DilJob;
static void dilate_slabs(void* c, i64 lo, i64 hi, int tid) {
    (void)tid;
    DilJob* j = (DilJob*)c;
    i64 dimsv[3] = {j->nx, j->ny, j->nz};
    i64 stride[3] = {j->ny * j->nz, j->nz, 1};
    for (i64 x = lo; x < hi; ++x)
        for (i64 y = 0; y < j->ny; ++y)
            for (i64 z = 0; z < j->nz; ++z) {
                i64 cc[3] = {x, y, z};
                i64 i = IDX3(x, y, z, j->ny, j->nz);
                uint8_t v = j->tmp[i];
                if (cc[j->axis] > 0) v |= j->tmp[i - stride[j->axis]];
                if (cc[j->axis] < dimsv[j->axis] - 1) v |= j->tmp[i + stride[j->axis]];
                j->bits[i] = v;
            }
}
static void dilate26(uint8_t* bits, i64 nx, i64 ny, i64 nz) {
    i64 n = nx * ny * nz;
    uint8_t* tmp = (uint8_t*)malloc((size_t)n);
    for (int axis = 0; axis < 3; ++axis) {
        memcpy(tmp, bits, (size_t)n);
        DilJob j = {bits, tmp, nx, ny, nz, axis};
        par_for(nx, dilate_slabs, &j);
    }
    free(tmp);
}

typedef struct {
    const void* vol; int is_f32; i64 plane; const float* tab; const uint8_t* vis; uint8_t* out;
    i64 counts[64];
} ClsJob;
static void classify_slabs(void* c, i64 lo, i64 hi, int tid) {
    ClsJob* j = (ClsJob*)c;
    i64 count = 0;
    for (i64 i = lo * j->plane; i < hi * j->plane; ++i) {
        uint8_t v = j->vis[quantize_f32(field_value(j->vol, j->is_f32, i, j->tab))];
        j->out[i] = v;
        count += v;
    }
    j->counts[tid] = count;
}

/* volume.py:379-391 + 394-396.  Returns the count of NON-dilated visible voxels. */
i64 or_classify(const void* vol, int is_f32, i64 nx, i64 ny, i64 nz, const float* lut,
                int dilate, uint8_t* out) {
    float tab[256];
    or_u8_field_table(tab);
    uint8_t vis[256];
    for (int b = 0; b < 256; ++b) vis[b] = lut[4 * b + 3] > 0.0f;
    ClsJob j;
    memset(&j, 0, sizeof j);
    j.vol = vol; j.is_f32 = is_f32; j.plane = ny * nz; j.tab = tab; j.vis = vis; j.out = out;
    int nt = par_for(nx, classify_slabs, &j);
    i64 count = 0;
    for (int t = 0; t < nt; ++t) count += j.counts[t];
    if (dilate) dilate26(out, nx, ny, nz);
    return count;
}

/* ------------------------------------------------------------------------------------ */
/* Morton codes: lbvh.py:25-66                                                           */
/* ------------------------------------------------------------------------------------ */

static uint64_t spread_bits(uint64_t v) {
    v = (v | (v << 16)) & 0x030000FFull;
    v = (v | (v << 8)) & 0x0300F00Full;
    v = (v | (v << 4)) & 0x030C30C3ull;
    v = (v | (v << 2)) & 0x09249249ull;
    return v;
}

uint32_t or_morton_encode(i64 x, i64 y, i64 z) {
    return (uint32_t)(spread_bits((uint64_t)x) | (spread_bits((uint64_t)y) << 1) |
                      (spread_bits((uint64_t)z) << 2));
}

/* ------------------------------------------------------------------------------------ */
/* flag_bricks: lbvh.py:83-102.  Brick (bx,by,bz) is voted iff any flag in              */
/* [b*bs, (b+1)*bs) clipped to dims; output in np.argwhere (C) order.                    */
/* Returns the count, or -count when cap is too small (nothing past cap written).        */
/* ------------------------------------------------------------------------------------ */
typedef struct { const uint8_t* bits; i64 nx, ny, nz, bs, nb[3]; uint8_t* vote; } VoteJob;
static void vote_slabs(void* c, i64 lo, i64 hi, int tid) {
    (void)tid;
    VoteJob* j = (VoteJob*)c;
    for (i64 bx = lo; bx < hi; ++bx)
        for (i64 by = 0; by < j->nb[1]; ++by)
            for (i64 bz = 0; bz < j->nb[2]; ++bz) {
                int any = 0;
                for (i64 x = bx * j->bs; x < imin64((bx + 1) * j->bs, j->nx) && !any; ++x)
                    for (i64 y = by * j->bs; y < imin64((by + 1) * j->bs, j->ny) && !any; ++y)
                        for (i64 z = bz * j->bs; z < imin64((bz + 1) * j->bs, j->nz); ++z)
                            if (j->bits[IDX3(x, y, z, j->ny, j->nz)]) { any = 1; break; }
                j->vote[IDX3(bx, by, bz, j->nb[1], j->nb[2])] = (uint8_t)any;
            }
}
i64 or_flag_bricks(const uint8_t* bits, i64 nx, i64 ny, i64 nz, i64 bs, int32_t* coords,
                   uint32_t* codes, i64 cap) {
    VoteJob j = {bits, nx, ny, nz, bs, {(nx + bs - 1) / bs, (ny + bs - 1) / bs, (nz + bs - 1) / bs},
                 NULL};
    i64 nbt = j.nb[0] * j.nb[1] * j.nb[2];
    j.vote = (uint8_t*)malloc((size_t)(nbt > 0 ? nbt : 1));
    par_for(j.nb[0], vote_slabs, &j);
    i64 cnt = 0;
    for (i64 bx = 0; bx < j.nb[0]; ++bx)
        for (i64 by = 0; by < j.nb[1]; ++by)
            for (i64 bz = 0; bz < j.nb[2]; ++bz) {
                if (!j.vote[IDX3(bx, by, bz, j.nb[1], j.nb[2])]) continue;
                if (cnt < cap) {
                    coords[3 * cnt] = (int32_t)bx;
                    coords[3 * cnt + 1] = (int32_t)by;
                    coords[3 * cnt + 2] = (int32_t)bz;
                    codes[cnt] = or_morton_encode(bx, by, bz);
                }
                cnt++;
            }
    free(j.vote);
    return cnt <= cap ? cnt : -cnt;
}

/* ------------------------------------------------------------------------------------ */
/* build_lbvh: lbvh.py:153-264 (Karras radix tree + refit)                               */
/* ------------------------------------------------------------------------------------ */

/* lbvh.py:153-164 */
static int common_prefix(const uint64_t* keys, i64 i, i64 j, i64 n) {
    if (j < 0 || j >= n) return -1;
    uint64_t x = keys[i] ^ keys[j];
    if (x == 0) return 64;
    return __builtin_clzll(x);
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

typedef struct { i64 key; i64 idx; } KeyIdx;
static int cmp_keyidx(const void* a, const void* b) {
    const KeyIdx* p = (const KeyIdx*)a; const KeyIdx* q = (const KeyIdx*)b;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    return p->idx < q->idx ? -1 : (p->idx > q->idx ? 1 : 0);
}

/* Outputs sized m = 2n-1 rows (lo/hi m*3, left/right/leaf_brick m) and sorted_coords n*3.
 * Returns the tree height (lbvh.py:128-144). */
i64 or_build_lbvh(const int32_t* coords, const uint32_t* codes, i64 n, i64 bs, i64 nx, i64 ny,
                  i64 nz, int32_t* lo, int32_t* hi, int32_t* left, int32_t* right,
                  int32_t* leaf_brick, int32_t* sorted_coords) {
    if (n == 0) return 0;
    i64 dims[3] = {nx, ny, nz};
    /* lbvh.py:226-229: keys = code<<32 | scan index, stable argsort (keys are unique) */
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n);
    for (i64 i = 0; i < n; ++i) keys[i] = ((uint64_t)codes[i] << 32) | (uint64_t)i;
    qsort(keys, (size_t)n, sizeof(uint64_t), cmp_u64);
    i64 m = 2 * n - 1;
    for (i64 i = 0; i < m; ++i) { left[i] = -1; right[i] = -1; leaf_brick[i] = -1; }
    for (i64 k = 0; k < n; ++k) {
        i64 src = (i64)(keys[k] & 0xffffffffull);
        for (int a = 0; a < 3; ++a) {
            int32_t c = coords[3 * src + a];
            sorted_coords[3 * k + a] = c;
            i64 l = (i64)c * bs;                       /* lbvh.py:231-232 */
            lo[3 * (n - 1 + k) + a] = (int32_t)l;
            hi[3 * (n - 1 + k) + a] = (int32_t)imin64(l + bs, dims[a]);
        }
        leaf_brick[n - 1 + k] = (int32_t)k;
    }
    i64 height = 1;
    if (n > 1) {
        i64* first = (i64*)malloc(sizeof(i64) * (n - 1));
        i64* last = (i64*)malloc(sizeof(i64) * (n - 1));
        /* lbvh.py:167-200 */
        for (i64 i = 0; i < n - 1; ++i) {
            int d = common_prefix(keys, i, i + 1, n) > common_prefix(keys, i, i - 1, n) ? 1 : -1;
            int delta_min = common_prefix(keys, i, i - d, n);
            i64 lmax = 2;
            while (common_prefix(keys, i, i + lmax * d, n) > delta_min) lmax *= 2;
            i64 length = 0;
            for (i64 t = lmax / 2; t >= 1; t /= 2)
                if (common_prefix(keys, i, i + (length + t) * d, n) > delta_min) length += t;
            i64 j = i + length * d;
            int delta_node = common_prefix(keys, i, j, n);
            i64 s = 0, t = length;
            while (1) {
                t = (t + 1) / 2;
                if (common_prefix(keys, i, i + (s + t) * d, n) > delta_node) s += t;
                if (t == 1) break;
            }
            i64 gamma = i + s * d + (d < 0 ? d : 0);
            i64 l0 = i < j ? i : j, h0 = i > j ? i : j;
            first[i] = l0;
            last[i] = h0;
            left[i] = (int32_t)(l0 == gamma ? (n - 1) + gamma : gamma);
            right[i] = (int32_t)(h0 == gamma + 1 ? (n - 1) + gamma + 1 : gamma + 1);
        }
        /* lbvh.py:248-249: refit children-before-parents (stable argsort of last-first) */
        KeyIdx* ord = (KeyIdx*)malloc(sizeof(KeyIdx) * (n - 1));
        for (i64 i = 0; i < n - 1; ++i) { ord[i].key = last[i] - first[i]; ord[i].idx = i; }
        qsort(ord, (size_t)(n - 1), sizeof(KeyIdx), cmp_keyidx);
        i64* hgt = (i64*)calloc((size_t)m, sizeof(i64));
        for (i64 k = n - 1; k < m; ++k) hgt[k] = 1;
        for (i64 k = 0; k < n - 1; ++k) {                 /* lbvh.py:203-213 */
            i64 i = ord[k].idx, l = left[i], r = right[i];
            for (int a = 0; a < 3; ++a) {
                lo[3 * i + a] = lo[3 * l + a] < lo[3 * r + a] ? lo[3 * l + a] : lo[3 * r + a];
                hi[3 * i + a] = hi[3 * l + a] > hi[3 * r + a] ? hi[3 * l + a] : hi[3 * r + a];
            }
            hgt[i] = 1 + (hgt[l] > hgt[r] ? hgt[l] : hgt[r]);
        }
        height = hgt[0];
        free(hgt); free(ord); free(first); free(last);
    }
    free(keys);
    return height;
}

/* ------------------------------------------------------------------------------------ */
/* SVT tables and queries: svt.py:40-131                                                 */
/* ------------------------------------------------------------------------------------ */

/* svt.py:40-57.  tables: (nbx,nby,nbz,bs+1,bs+1,bs+1) uint32, zero border, padding zero. */
void or_svt_build(const uint8_t* bits, i64 nx, i64 ny, i64 nz, i64 bs, uint32_t* tables) {
    i64 nb[3] = {(nx + bs - 1) / bs, (ny + bs - 1) / bs, (nz + bs - 1) / bs};
    i64 t = bs + 1, tb = t * t * t;
    for (i64 bx = 0; bx < nb[0]; ++bx)
        for (i64 by = 0; by < nb[1]; ++by)
            for (i64 bz = 0; bz < nb[2]; ++bz) {
                uint32_t* T = tables + ((bx * nb[1] + by) * nb[2] + bz) * tb;
                memset(T, 0, sizeof(uint32_t) * tb);
                for (i64 i = 1; i <= bs; ++i)
                    for (i64 j = 1; j <= bs; ++j)
                        for (i64 k = 1; k <= bs; ++k) {
                            i64 x = bx * bs + i - 1, y = by * bs + j - 1, z = bz * bs + k - 1;
                            uint32_t v = (x < nx && y < ny && z < nz) ? bits[IDX3(x, y, z, ny, nz)] : 0;
                            /* 3-d inclusion-exclusion == the reference's three cumsums */
                            T[(i * t + j) * t + k] = v + T[((i - 1) * t + j) * t + k] +
                                                     T[(i * t + j - 1) * t + k] + T[(i * t + j) * t + k - 1] -
                                                     T[((i - 1) * t + j - 1) * t + k] -
                                                     T[((i - 1) * t + j) * t + k - 1] -
                                                     T[(i * t + j - 1) * t + k - 1] +
                                                     T[((i - 1) * t + j - 1) * t + k - 1];
                        }
            }
}

/* svt.py:65-90; box in/out as lo[3], hi[3]; clipped to dims first (svt.py:61-63) */
i64 or_box_count(const uint32_t* tables, i64 nx, i64 ny, i64 nz, i64 bs, const i64* blo,
                 const i64* bhi) {
    i64 dims[3] = {nx, ny, nz};
    i64 lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = imax64(blo[a], 0);
        hi[a] = imin64(bhi[a], dims[a]);
        if (lo[a] >= hi[a]) return 0;
    }
    i64 nb[3] = {(nx + bs - 1) / bs, (ny + bs - 1) / bs, (nz + bs - 1) / bs};
    i64 t = bs + 1, tb = t * t * t;
    i64 total = 0;
    for (i64 bx = lo[0] / bs; bx <= (hi[0] - 1) / bs; ++bx)
        for (i64 by = lo[1] / bs; by <= (hi[1] - 1) / bs; ++by)
            for (i64 bz = lo[2] / bs; bz <= (hi[2] - 1) / bs; ++bz) {
                const uint32_t* T = tables + ((bx * nb[1] + by) * nb[2] + bz) * tb;
                i64 b[3] = {bx, by, bz}, l[3], h[3];
                for (int a = 0; a < 3; ++a) {
                    l[a] = imin64(imax64(lo[a] - b[a] * bs, 0), bs);
                    h[a] = imin64(imax64(hi[a] - b[a] * bs, 0), bs);
                }
                for (int sx = 0; sx < 2; ++sx)
                    for (int sy = 0; sy < 2; ++sy)
                        for (int sz = 0; sz < 2; ++sz) {
                            i64 ix = sx ? l[0] : h[0], iy = sy ? l[1] : h[1], iz = sz ? l[2] : h[2];
                            i64 sign = ((sx + sy + sz) & 1) ? -1 : 1;
                            total += sign * (i64)T[(ix * t + iy) * t + iz];
                        }
            }
    return total;
}

/* svt.py:100-131: per-axis binary search on monotone slab counts.  Returns 0 for None. */
int or_shrink_svt(const uint32_t* tables, i64 nx, i64 ny, i64 nz, i64 bs, const i64* blo,
                  const i64* bhi, i64* olo, i64* ohi) {
    i64 dims[3] = {nx, ny, nz};
    i64 lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = imax64(blo[a], 0);
        hi[a] = imin64(bhi[a], dims[a]);
        if (lo[a] >= hi[a]) return 0;
    }
    if (or_box_count(tables, nx, ny, nz, bs, lo, hi) == 0) return 0;
    for (int axis = 0; axis < 3; ++axis) {
        i64 a0 = lo[axis], a1 = hi[axis];
        i64 ql[3], qh[3];
        i64 low = a0 + 1, high = a1;
        while (low < high) {
            i64 mid = (low + high) / 2;
            memcpy(ql, lo, sizeof ql); memcpy(qh, hi, sizeof qh);
            ql[axis] = a0; qh[axis] = mid;
            if (or_box_count(tables, nx, ny, nz, bs, ql, qh) > 0) high = mid; else low = mid + 1;
        }
        olo[axis] = low - 1;
        low = a0; high = a1 - 1;
        while (low < high) {
            i64 mid = (low + high + 1) / 2;
            memcpy(ql, lo, sizeof ql); memcpy(qh, hi, sizeof qh);
            ql[axis] = mid; qh[axis] = a1;
            if (or_box_count(tables, nx, ny, nz, bs, ql, qh) > 0) low = mid; else high = mid - 1;
        }
        ohi[axis] = low + 1;
    }
    return 1;
}

/* Exact tight box of the flags in [blo, bhi) by direct scan; equal to shrink_to_occupied
 * (pinned by tests/test_oracle_golden.py::test_shrink_direct_equals_svt). */
int or_tight_box(const uint8_t* bits, i64 nx, i64 ny, i64 nz, const i64* blo, const i64* bhi,
                 i64* olo, i64* ohi) {
    i64 dims[3] = {nx, ny, nz};
    i64 lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = imax64(blo[a], 0);
        hi[a] = imin64(bhi[a], dims[a]);
        if (lo[a] >= hi[a]) return 0;
    }
    i64 mn[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, mx[3] = {-1, -1, -1};
    for (i64 x = lo[0]; x < hi[0]; ++x)
        for (i64 y = lo[1]; y < hi[1]; ++y) {
            const uint8_t* row = bits + IDX3(x, y, 0, ny, nz);
            for (i64 z = lo[2]; z < hi[2]; ++z)
                if (row[z]) {
                    if (x < mn[0]) mn[0] = x;
                    if (x > mx[0]) mx[0] = x;
                    if (y < mn[1]) mn[1] = y;
                    if (y > mx[1]) mx[1] = y;
                    if (z < mn[2]) mn[2] = z;
                    if (z > mx[2]) mx[2] = z;
                }
        }
    if (mx[0] < 0) return 0;
    for (int a = 0; a < 3; ++a) { olo[a] = mn[a]; ohi[a] = mx[a] + 1; }
    return 1;
}

/* svt.py:161-167 (_macro_from_bits): cell occupied iff any flag in the (clipped) cell. */
void or_macro_grid(const uint8_t* bits, i64 nx, i64 ny, i64 nz, i64 cs, uint8_t* occ) {
    i64 nc[3] = {(nx + cs - 1) / cs, (ny + cs - 1) / cs, (nz + cs - 1) / cs};
    memset(occ, 0, (size_t)(nc[0] * nc[1] * nc[2]));
    for (i64 x = 0; x < nx; ++x)
        for (i64 y = 0; y < ny; ++y)
            for (i64 z = 0; z < nz; ++z)
                if (bits[IDX3(x, y, z, ny, nz)]) occ[IDX3(x / cs, y / cs, z / cs, nc[1], nc[2])] = 1;
}

/* ------------------------------------------------------------------------------------ */
/* Cell boxes: kdtree.py:285-320 (precompute_cell_boxes).  Rows sorted by cell Morton     */
/* code; unoccupied rows hold the reference's placeholder (full unclipped cell).          */
/* ------------------------------------------------------------------------------------ */
typedef struct { uint32_t code; i64 cell; } CodeCell;
static int cmp_codecell(const void* a, const void* b) {
    uint32_t x = ((const CodeCell*)a)->code, y = ((const CodeCell*)b)->code;
    return x < y ? -1 : (x > y ? 1 : 0);
}

void or_cell_boxes(const uint8_t* bits, i64 nx, i64 ny, i64 nz, i64 cs, uint32_t* codes,
                   int32_t* coords, int32_t* lo, int32_t* hi, uint8_t* occupied) {
    i64 nc[3] = {(nx + cs - 1) / cs, (ny + cs - 1) / cs, (nz + cs - 1) / cs};
    i64 ncell = nc[0] * nc[1] * nc[2];
    CodeCell* cc = (CodeCell*)malloc(sizeof(CodeCell) * ncell);
    for (i64 c = 0; c < ncell; ++c) {
        i64 cx = c / (nc[1] * nc[2]), cy = (c / nc[2]) % nc[1], cz = c % nc[2];
        cc[c].code = or_morton_encode(cx, cy, cz);
        cc[c].cell = c;
    }
    qsort(cc, (size_t)ncell, sizeof(CodeCell), cmp_codecell);
    for (i64 r = 0; r < ncell; ++r) {
        i64 c = cc[r].cell;
        i64 cxyz[3] = {c / (nc[1] * nc[2]), (c / nc[2]) % nc[1], c % nc[2]};
        i64 mn[3] = {cs, cs, cs}, mx[3] = {-1, -1, -1};
        for (i64 i = 0; i < cs; ++i)
            for (i64 j = 0; j < cs; ++j)
                for (i64 k = 0; k < cs; ++k) {
                    i64 x = cxyz[0] * cs + i, y = cxyz[1] * cs + j, z = cxyz[2] * cs + k;
                    if (x >= nx || y >= ny || z >= nz || !bits[IDX3(x, y, z, ny, nz)]) continue;
                    i64 l[3] = {i, j, k};
                    for (int a = 0; a < 3; ++a) {
                        if (l[a] < mn[a]) mn[a] = l[a];
                        if (l[a] > mx[a]) mx[a] = l[a];
                    }
                }
        int occ = mx[0] >= 0;
        codes[r] = cc[r].code;
        occupied[r] = (uint8_t)occ;
        for (int a = 0; a < 3; ++a) {
            coords[3 * r + a] = (int32_t)cxyz[a];
            /* argmax of an all-false row is 0 -> placeholder [c*cs, c*cs + cs) */
            lo[3 * r + a] = (int32_t)(cxyz[a] * cs + (occ ? mn[a] : 0));
            hi[3 * r + a] = (int32_t)(cxyz[a] * cs + (occ ? mx[a] : cs - 1) + 1);
        }
    }
    free(cc);
}

/* ------------------------------------------------------------------------------------ */
/* k-d tree builders: kdtree.py:148-498                                                  */
/* ------------------------------------------------------------------------------------ */
typedef struct { i64 lo[3], hi[3]; } Box;

static i64 box_volume(const Box* b) {
    return (b->hi[0] - b->lo[0]) * (b->hi[1] - b->lo[1]) * (b->hi[2] - b->lo[2]);
}

typedef struct {
    const uint8_t* bits;
    i64 dims[3];
    int mode_deep;        /* 0 shallow, 1 deep */
    i64 mls;              /* -1 = None */
    int binned;
    i64 bins, cs;
    i64 root_vol;
    /* binned cell data (kdtree.py:285-320), indexed by C-order cell id */
    i64 nc[3];
    uint8_t* cocc;
    int32_t* clo;
    int32_t* chi;
    /* output rows (DFS preorder, kdtree.py:412-419) */
    i64 n, cap;
    int32_t *lo, *hi, *plane, *left, *right;
    int8_t* axis;
} KdCtx;

static i64 emit(KdCtx* k, const Box* b, int axis, i64 plane) {
    if (k->n == k->cap) {
        k->cap = k->cap ? 2 * k->cap : 1024;
        k->lo = (int32_t*)realloc(k->lo, sizeof(int32_t) * 3 * k->cap);
        k->hi = (int32_t*)realloc(k->hi, sizeof(int32_t) * 3 * k->cap);
        k->plane = (int32_t*)realloc(k->plane, sizeof(int32_t) * k->cap);
        k->left = (int32_t*)realloc(k->left, sizeof(int32_t) * k->cap);
        k->right = (int32_t*)realloc(k->right, sizeof(int32_t) * k->cap);
        k->axis = (int8_t*)realloc(k->axis, sizeof(int8_t) * k->cap);
    }
    i64 i = k->n++;
    for (int a = 0; a < 3; ++a) { k->lo[3 * i + a] = (int32_t)b->lo[a]; k->hi[3 * i + a] = (int32_t)b->hi[a]; }
    k->axis[i] = (int8_t)axis;
    k->plane[i] = (int32_t)plane;
    k->left[i] = -1;
    k->right[i] = -1;
    return i;
}

/* kdtree.py:421-424 */
static int halted(const KdCtx* k, i64 vol) {
    if (!k->mode_deep) return vol * 10 <= k->root_vol;
    return vol <= 512;
}

/* kdtree.py:156-221 (_axis_sweep, _side_volumes, _sweep_search) over the region bits of
 * box.  Returns 1 and fills (axis, cut k, cost, left/right boxes or has_l/has_r = 0). */
static int sweep_search(const KdCtx* k, const Box* box, int* o_axis, i64* o_k, i64* o_cost,
                        Box* o_l, int* has_l, Box* o_r, int* has_r) {
    const i64 FAR = (i64)1 << 60;
    i64 e[3] = {box->hi[0] - box->lo[0], box->hi[1] - box->lo[1], box->hi[2] - box->lo[2]};
    i64 ny = k->dims[1], nz = k->dims[2];
    /* projections (kdtree.py:196): pxy[x][y], pxz[x][z], pyz[y][z] */
    uint8_t* pxy = (uint8_t*)calloc((size_t)(e[0] * e[1]), 1);
    uint8_t* pxz = (uint8_t*)calloc((size_t)(e[0] * e[2]), 1);
    uint8_t* pyz = (uint8_t*)calloc((size_t)(e[1] * e[2]), 1);
    for (i64 x = 0; x < e[0]; ++x)
        for (i64 y = 0; y < e[1]; ++y) {
            const uint8_t* row = k->bits + IDX3(box->lo[0] + x, box->lo[1] + y, box->lo[2], ny, nz);
            for (i64 z = 0; z < e[2]; ++z)
                if (row[z]) { pxy[x * e[1] + y] = 1; pxz[x * e[2] + z] = 1; pyz[y * e[2] + z] = 1; }
        }
    /* rows order per axis: a=0 (x; y from pxy, z from pxz); a=1 (y; x from pxy^T, z from
     * pyz); a=2 (z; x from pxz^T, y from pyz^T) -- kdtree.py:198-204 */
    static const int ROWS_TO_XYZ[3][3] = {{0, 1, 2}, {1, 0, 2}, {1, 2, 0}};
    int found = 0;
    i64 best_cost = 0;
    for (int a = 0; a < 3; ++a) {
        i64 ea = e[a];
        if (ea < 2) continue;
        i64 e1 = a == 0 ? e[1] : e[0];     /* columns of pa */
        i64 e2 = a == 2 ? e[1] : e[2];     /* columns of pb */
        i64* F = (i64*)malloc(sizeof(i64) * 3 * ea);
        i64* L = (i64*)malloc(sizeof(i64) * 3 * ea);
        for (i64 s = 0; s < ea; ++s) {
            i64 f1 = -1, l1 = -1, f2 = -1, l2 = -1;
            for (i64 c = 0; c < e1; ++c) {
                uint8_t v = a == 0 ? pxy[s * e[1] + c] : (a == 1 ? pxy[c * e[1] + s] : pxz[c * e[2] + s]);
                if (v) { if (f1 < 0) f1 = c; l1 = c; }
            }
            for (i64 c = 0; c < e2; ++c) {
                uint8_t v = a == 0 ? pxz[s * e[2] + c] : (a == 1 ? pyz[s * e[2] + c] : pyz[c * e[2] + s]);
                if (v) { if (f2 < 0) f2 = c; l2 = c; }
            }
            int ok = f1 >= 0;
            F[0 * ea + s] = ok ? s : FAR;  L[0 * ea + s] = ok ? s : -1;
            F[1 * ea + s] = ok ? f1 : FAR; L[1 * ea + s] = ok ? l1 : -1;
            F[2 * ea + s] = ok ? f2 : FAR; L[2 * ea + s] = ok ? l2 : -1;
        }
        i64 *pl = (i64*)malloc(sizeof(i64) * 3 * ea), *ph = (i64*)malloc(sizeof(i64) * 3 * ea);
        i64 *sl = (i64*)malloc(sizeof(i64) * 3 * ea), *sh = (i64*)malloc(sizeof(i64) * 3 * ea);
        for (int r = 0; r < 3; ++r) {
            for (i64 s = 0; s < ea; ++s) {
                pl[r * ea + s] = s ? imin64(pl[r * ea + s - 1], F[r * ea + s]) : F[r * ea + s];
                ph[r * ea + s] = s ? imax64(ph[r * ea + s - 1], L[r * ea + s]) : L[r * ea + s];
            }
            for (i64 s = ea - 1; s >= 0; --s) {
                sl[r * ea + s] = s < ea - 1 ? imin64(sl[r * ea + s + 1], F[r * ea + s]) : F[r * ea + s];
                sh[r * ea + s] = s < ea - 1 ? imax64(sh[r * ea + s + 1], L[r * ea + s]) : L[r * ea + s];
            }
        }
        /* cost[k-1] = vol(pre[k-1]) + vol(suf[k]), k = 1..ea-1; first minimum */
        i64 bk = -1, bc = 0;
        for (i64 kk = 1; kk < ea; ++kk) {
            i64 vl = 0, vr = 0;
            if (ph[0 * ea + kk - 1] >= 0)
                vl = (ph[kk - 1] - pl[kk - 1] + 1) * (ph[ea + kk - 1] - pl[ea + kk - 1] + 1) *
                     (ph[2 * ea + kk - 1] - pl[2 * ea + kk - 1] + 1);
            if (sh[0 * ea + kk] >= 0)
                vr = (sh[kk] - sl[kk] + 1) * (sh[ea + kk] - sl[ea + kk] + 1) *
                     (sh[2 * ea + kk] - sl[2 * ea + kk] + 1);
            i64 c = vl + vr;
            if (bk < 0 || c < bc) { bk = kk; bc = c; }
        }
        if (!(found && bc >= best_cost)) {  /* kdtree.py:212-213: strict < across axes */
            found = 1;
            best_cost = bc;
            *o_axis = a;
            *o_k = bk;
            *o_cost = bc;
            const int* rows = ROWS_TO_XYZ[a];
            *has_l = ph[0 * ea + bk - 1] >= 0;
            if (*has_l)
                for (int i = 0; i < 3; ++i) {
                    o_l->lo[i] = box->lo[i] + pl[rows[i] * ea + bk - 1];
                    o_l->hi[i] = box->lo[i] + ph[rows[i] * ea + bk - 1] + 1;
                }
            *has_r = sh[0 * ea + bk] >= 0;
            if (*has_r)
                for (int i = 0; i < 3; ++i) {
                    o_r->lo[i] = box->lo[i] + sl[rows[i] * ea + bk];
                    o_r->hi[i] = box->lo[i] + sh[rows[i] * ea + bk] + 1;
                }
        }
        free(F); free(L); free(pl); free(ph); free(sl); free(sh);
    }
    free(pxy); free(pxz); free(pyz);
    return found;
}

/* kdtree.py:323-343 (_cells_reduce).  The Morton-range prefilter in the reference is an
 * acceleration only: Morton codes are monotone per axis, so every cell with coords in
 * [clo, chi] lies in [code(clo), code(chi)].  The selection is therefore "occupied cells
 * with clo <= coords <= chi"; union of their boxes, clipped back to the region. */
static int cells_reduce(const KdCtx* k, const Box* region, Box* out) {
    i64 clo[3], chi[3];
    for (int a = 0; a < 3; ++a) {
        clo[a] = imax64(floordiv(region->lo[a], k->cs), 0);
        chi[a] = imin64(floordiv(region->hi[a] - 1, k->cs), k->nc[a] - 1);
        if (clo[a] > chi[a]) return 0;
    }
    i64 mn[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, mx[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
    int any = 0;
    for (i64 cx = clo[0]; cx <= chi[0]; ++cx)
        for (i64 cy = clo[1]; cy <= chi[1]; ++cy)
            for (i64 cz = clo[2]; cz <= chi[2]; ++cz) {
                i64 c = IDX3(cx, cy, cz, k->nc[1], k->nc[2]);
                if (!k->cocc[c]) continue;
                any = 1;
                for (int a = 0; a < 3; ++a) {
                    if (k->clo[3 * c + a] < mn[a]) mn[a] = k->clo[3 * c + a];
                    if (k->chi[3 * c + a] > mx[a]) mx[a] = k->chi[3 * c + a];
                }
            }
    if (!any) return 0;
    for (int a = 0; a < 3; ++a) {
        out->lo[a] = imax64(mn[a], region->lo[a]);
        out->hi[a] = imin64(mx[a], region->hi[a]);
        if (out->lo[a] >= out->hi[a]) return 0;
    }
    return 1;
}

/* kdtree.py:346-350: float64 snapping, deduped and sorted. */
int or_snapped_positions(i64 lo, i64 hi, i64 bins, i64 cs, i64* out) {
    i64 extent = hi - lo;
    double step = (double)extent / (double)bins;
    int n = 0;
    for (i64 j = 1; j < bins; ++j) {
        double raw = (double)lo + (double)j * step;
        i64 p = (i64)floor(raw / (double)cs + 0.5) * cs;
        if (!(lo < p && p < hi)) continue;
        int dup = 0;
        for (int q = 0; q < n; ++q) if (out[q] == p) dup = 1;
        if (!dup) out[n++] = p;
    }
    for (int i = 1; i < n; ++i)            /* sorted() */
        for (int j = i; j > 0 && out[j - 1] > out[j]; --j) { i64 t = out[j]; out[j] = out[j - 1]; out[j - 1] = t; }
    return n;
}

/* kdtree.py:353-368 */
static int binned_search(const KdCtx* k, const Box* box, int* o_axis, i64* o_pos, i64* o_cost,
                         Box* o_l, int* has_l, Box* o_r, int* has_r) {
    int found = 0;
    i64 best = 0;
    i64 cand[64];
    for (int a = 0; a < 3; ++a) {
        int nc = or_snapped_positions(box->lo[a], box->hi[a], k->bins, k->cs, cand);
        for (int q = 0; q < nc; ++q) {
            i64 p = cand[q];
            Box lr = *box, rr = *box, lb, rb;
            lr.hi[a] = p;
            rr.lo[a] = p;
            int hl = cells_reduce(k, &lr, &lb), hr = cells_reduce(k, &rr, &rb);
            i64 cost = (hl ? box_volume(&lb) : 0) + (hr ? box_volume(&rb) : 0);
            if (!found || cost < best) {
                found = 1;
                best = cost;
                *o_axis = a; *o_pos = p; *o_cost = cost;
                *has_l = hl; if (hl) *o_l = lb;
                *has_r = hr; if (hr) *o_r = rb;
            }
        }
    }
    return found;
}

static int tight(const KdCtx* k, const Box* b, Box* out) {
    return or_tight_box(k->bits, k->dims[0], k->dims[1], k->dims[2], b->lo, b->hi, out->lo, out->hi);
}

/* kdtree.py:469-484 */
static i64 kd_build_rec(KdCtx* k, const Box* box) {
    int axis = -1, has_l = 0, has_r = 0, split = 0;
    i64 pos = 0, cost = 0;
    Box lb, rb;
    i64 vol = box_volume(box);
    if (!halted(k, vol)) {                                   /* kdtree.py:426-439 */
        if (k->binned) {
            if (binned_search(k, box, &axis, &pos, &cost, &lb, &has_l, &rb, &has_r) && cost < vol) split = 1;
        } else {
            i64 kk = 0;
            if (sweep_search(k, box, &axis, &kk, &cost, &lb, &has_l, &rb, &has_r) && cost < vol) {
                split = 1;
                pos = box->lo[axis] + kk;
            }
        }
    }
    if (!split && k->mls >= 0) {                             /* kdtree.py:441-467 */
        i64 ext[3] = {box->hi[0] - box->lo[0], box->hi[1] - box->lo[1], box->hi[2] - box->lo[2]};
        i64 mx = imax64(ext[0], imax64(ext[1], ext[2]));
        if (mx > k->mls) {
            axis = ext[0] == mx ? 0 : (ext[1] == mx ? 1 : 2);  /* np.argmax: first max */
            i64 lo = box->lo[axis], hi = box->hi[axis];
            pos = lo + ext[axis] / 2;
            if (k->binned) {
                i64 cs = k->cs;
                i64 first = (floordiv(lo, cs) + 1) * cs;
                i64 last = floordiv(hi - 1, cs) * cs;
                if (first <= last) {
                    i64 snapped = (i64)floor((double)pos / (double)cs + 0.5) * cs;
                    pos = imin64(imax64(snapped, first), last);
                }
            }
            Box lr = *box, rr = *box;
            lr.hi[axis] = pos;
            rr.lo[axis] = pos;
            if (k->binned) {
                has_l = cells_reduce(k, &lr, &lb);
                has_r = cells_reduce(k, &rr, &rb);
            } else {
                has_l = tight(k, &lr, &lb);
                has_r = tight(k, &rr, &rb);
            }
            split = 1;
        }
    }
    if (!split) {
        if (k->binned) {                                       /* kdtree.py:474 */
            Box leaf;
            if (!tight(k, box, &leaf)) return -1;
            return emit(k, &leaf, -1, -1);
        }
        return emit(k, box, -1, -1);
    }
    i64 i = emit(k, box, axis, pos);
    i64 li = has_l ? kd_build_rec(k, &lb) : -1;
    i64 ri = has_r ? kd_build_rec(k, &rb) : -1;
    k->left[i] = (int32_t)li;
    k->right[i] = (int32_t)ri;
    return i;
}

/* kdtree.py:387-498.  Returns a heap-allocated result; free with or_kd_free. */
typedef struct {
    i64 n;
    i64 root;
    int32_t *lo, *hi, *plane, *left, *right;
    int8_t* axis;
} KdResult;

KdResult* or_kd_build(const uint8_t* bits, i64 nx, i64 ny, i64 nz, int mode_deep, i64 mls,
                      int binned, i64 bins, i64 cs) {
    KdCtx k;
    memset(&k, 0, sizeof k);
    k.bits = bits;
    k.dims[0] = nx; k.dims[1] = ny; k.dims[2] = nz;
    k.mode_deep = mode_deep; k.mls = mls; k.binned = binned; k.bins = bins; k.cs = cs;
    KdResult* res = (KdResult*)calloc(1, sizeof(KdResult));
    res->root = -1;
    Box full = {{0, 0, 0}, {nx, ny, nz}}, root;
    if (!tight(&k, &full, &root)) return res;              /* kdtree.py:398-400 */
    k.root_vol = box_volume(&root);
    if (binned) {
        k.nc[0] = (nx + cs - 1) / cs; k.nc[1] = (ny + cs - 1) / cs; k.nc[2] = (nz + cs - 1) / cs;
        i64 ncell = k.nc[0] * k.nc[1] * k.nc[2];
        k.cocc = (uint8_t*)calloc((size_t)ncell, 1);
        k.clo = (int32_t*)malloc(sizeof(int32_t) * 3 * ncell);
        k.chi = (int32_t*)malloc(sizeof(int32_t) * 3 * ncell);
        for (i64 c = 0; c < ncell; ++c) {
            i64 cx = c / (k.nc[1] * k.nc[2]), cy = (c / k.nc[2]) % k.nc[1], cz = c % k.nc[2];
            Box cell = {{cx * cs, cy * cs, cz * cs}, {(cx + 1) * cs, (cy + 1) * cs, (cz + 1) * cs}}, t;
            if (tight(&k, &cell, &t)) {
                k.cocc[c] = 1;
                for (int a = 0; a < 3; ++a) { k.clo[3 * c + a] = (int32_t)t.lo[a]; k.chi[3 * c + a] = (int32_t)t.hi[a]; }
            }
        }
    }
    i64 r = kd_build_rec(&k, &root);
    free(k.cocc); free(k.clo); free(k.chi);
    if (r < 0) {
        free(k.lo); free(k.hi); free(k.plane); free(k.left); free(k.right); free(k.axis);
        return res;
    }
    res->n = k.n; res->root = r;
    res->lo = k.lo; res->hi = k.hi; res->plane = k.plane; res->left = k.left; res->right = k.right; res->axis = k.axis;
    return res;
}

void or_kd_copy(const KdResult* r, int32_t* lo, int32_t* hi, int8_t* axis, int32_t* plane,
                int32_t* left, int32_t* right) {
    if (r->n == 0) return;
    memcpy(lo, r->lo, sizeof(int32_t) * 3 * r->n);
    memcpy(hi, r->hi, sizeof(int32_t) * 3 * r->n);
    memcpy(axis, r->axis, (size_t)r->n);
    memcpy(plane, r->plane, sizeof(int32_t) * r->n);
    memcpy(left, r->left, sizeof(int32_t) * r->n);
    memcpy(right, r->right, sizeof(int32_t) * r->n);
}

i64 or_kd_count(const KdResult* r) { return r->n; }
i64 or_kd_root(const KdResult* r) { return r->root; }

void or_kd_free(KdResult* r) {
    if (!r) return;
    free(r->lo); free(r->hi); free(r->plane); free(r->left); free(r->right); free(r->axis);
    free(r);
}

/* ------------------------------------------------------------------------------------ */
/* Renderer: render.py:196-911                                                            */
/* ------------------------------------------------------------------------------------ */
#define R_FAR 1e300

typedef struct {
    double ox, oy, oz, ix, iy, iz, dx, dy, dz;
    int zx, zy, zz;
} RaySt;

/* render.py:196-240 */
static int slab(const RaySt* r, double lx, double ly, double lz, double hx, double hy, double hz,
                double* t0, double* t1) {
    double tmin = -R_FAR, tmax = R_FAR, ta, tb;
    if (r->zx) { if (r->ox < lx || r->ox >= hx) return 0; }
    else {
        ta = (lx - r->ox) * r->ix; tb = (hx - r->ox) * r->ix;
        if (ta > tb) { double t = ta; ta = tb; tb = t; }
        if (ta > tmin) tmin = ta;
        if (tb < tmax) tmax = tb;
    }
    if (r->zy) { if (r->oy < ly || r->oy >= hy) return 0; }
    else {
        ta = (ly - r->oy) * r->iy; tb = (hy - r->oy) * r->iy;
        if (ta > tb) { double t = ta; ta = tb; tb = t; }
        if (ta > tmin) tmin = ta;
        if (tb < tmax) tmax = tb;
    }
    if (r->zz) { if (r->oz < lz || r->oz >= hz) return 0; }
    else {
        ta = (lz - r->oz) * r->iz; tb = (hz - r->oz) * r->iz;
        if (ta > tb) { double t = ta; ta = tb; tb = t; }
        if (ta > tmin) tmin = ta;
        if (tb < tmax) tmax = tb;
    }
    if (tmax <= tmin) return 0;
    *t0 = tmin; *t1 = tmax;
    return 1;
}

/* render.py:273-287 */
static void ray_setup(RaySt* r, const double* o, const double* d) {
    r->ox = o[0]; r->oy = o[1]; r->oz = o[2];
    r->dx = d[0]; r->dy = d[1]; r->dz = d[2];
    r->zx = d[0] == 0.0; r->zy = d[1] == 0.0; r->zz = d[2] == 0.0;
    r->ix = r->zx ? 0.0 : 1.0 / d[0];
    r->iy = r->zy ? 0.0 : 1.0 / d[1];
    r->iz = r->zz ? 0.0 : 1.0 / d[2];
}

typedef struct { double* t; i64 n, cap; } SegBuf;
static void seg_push(SegBuf* s, double a, double b) {
    if (s->n == s->cap) { s->cap = s->cap ? 2 * s->cap : 32; s->t = (double*)realloc(s->t, sizeof(double) * 2 * s->cap); }
    s->t[2 * s->n] = a; s->t[2 * s->n + 1] = b; s->n++;
}

/* render.py:243-270 */
static i64 sort_merge(double* seg, i64 m) {
    for (i64 i = 1; i < m; ++i) {
        double a0 = seg[2 * i], a1 = seg[2 * i + 1];
        i64 j = i - 1;
        while (j >= 0 && seg[2 * j] > a0) { seg[2 * j + 2] = seg[2 * j]; seg[2 * j + 3] = seg[2 * j + 1]; j--; }
        seg[2 * j + 2] = a0; seg[2 * j + 3] = a1;
    }
    i64 w = 0;
    for (i64 i = 0; i < m; ++i) {
        double t0 = seg[2 * i], t1 = seg[2 * i + 1];
        if (t1 <= t0) continue;
        if (w > 0 && t0 <= seg[2 * w - 1]) { if (t1 > seg[2 * w - 1]) seg[2 * w - 1] = t1; }
        else { seg[2 * w] = t0; seg[2 * w + 1] = t1; w++; }
    }
    return w;
}

typedef struct {
    int kind;                   /* 0 naive 1 grid 2 lbvh 3 kd 4 hybrid */
    i64 nx, ny, nz;
    /* grid */
    const uint8_t* occ; i64 ncx, ncy, ncz; double cs;
    /* trees (lbvh: axis = NULL, leaf iff left < 0) */
    const int32_t *lo, *hi, *left, *right, *plane;
    const int8_t* axis;
    i64 root;
} Index;

/* render.py:305-378 */
static void dda_runs(const RaySt* r, const Index* ix, double t_in, double t_out, SegBuf* out) {
    i64 ncx = ix->ncx, ncy = ix->ncy, ncz = ix->ncz;
    double cs = ix->cs;
    double px = r->ox + t_in * r->dx, py = r->oy + t_in * r->dy, pz = r->oz + t_in * r->dz;
    i64 cx = (i64)floor(px / cs), cy = (i64)floor(py / cs), cz = (i64)floor(pz / cs);
    if (cx < 0) cx = 0;
    if (cy < 0) cy = 0;
    if (cz < 0) cz = 0;
    if (cx > ncx - 1) cx = ncx - 1;
    if (cy > ncy - 1) cy = ncy - 1;
    if (cz > ncz - 1) cz = ncz - 1;
    int sx = r->zx ? 0 : (r->ix > 0.0 ? 1 : -1);
    int sy = r->zy ? 0 : (r->iy > 0.0 ? 1 : -1);
    int sz = r->zz ? 0 : (r->iz > 0.0 ? 1 : -1);
    double tnx = sx == 0 ? R_FAR : ((double)(cx + (sx > 0)) * cs - r->ox) * r->ix;
    double tny = sy == 0 ? R_FAR : ((double)(cy + (sy > 0)) * cs - r->oy) * r->iy;
    double tnz = sz == 0 ? R_FAR : ((double)(cz + (sz > 0)) * cs - r->oz) * r->iz;
    int open_run = 0;
    double run_t0 = 0.0, tcur = t_in;
    i64 max_steps = ncx + ncy + ncz + 3;
    for (i64 step = 0; step < max_steps; ++step) {
        double tn = tnx;
        if (tny < tn) tn = tny;
        if (tnz < tn) tn = tnz;
        if (ix->occ[IDX3(cx, cy, cz, ncy, ncz)]) {
            if (!open_run) { open_run = 1; run_t0 = tcur; }
        } else if (open_run) {
            seg_push(out, run_t0, tcur);
            open_run = 0;
        }
        if (tn >= t_out) break;
        if (tnx == tn) { cx += sx; tnx = ((double)(cx + (sx > 0)) * cs - r->ox) * r->ix; }
        if (tny == tn) { cy += sy; tny = ((double)(cy + (sy > 0)) * cs - r->oy) * r->iy; }
        if (tnz == tn) { cz += sz; tnz = ((double)(cz + (sz > 0)) * cs - r->oz) * r->iz; }
        tcur = tn;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= ncx || cy >= ncy || cz >= ncz) break;
    }
    if (open_run) seg_push(out, run_t0, t_out);
}

static int node_slab(const RaySt* r, const Index* ix, i64 i, double* a, double* b) {
    const int32_t *l = ix->lo + 3 * i, *h = ix->hi + 3 * i;
    return slab(r, (double)l[0], (double)l[1], (double)l[2], (double)h[0], (double)h[1], (double)h[2], a, b);
}

/* render.py:404-504 (leaf intervals, before _sort_merge) */
static void bvh_leaves(const RaySt* r, const Index* ix, double tmin, double tmax, SegBuf* out,
                       i64* stk, double* sa, double* sb) {
    double a, b;
    i64 sp = 0;
    if (node_slab(r, ix, ix->root, &a, &b)) {
        a = a > tmin ? a : tmin;
        b = b < tmax ? b : tmax;
        if (b > a) { stk[0] = ix->root; sa[0] = a; sb[0] = b; sp = 1; }
    }
    while (sp > 0) {
        sp--;
        i64 i = stk[sp];
        double t0 = sa[sp], t1 = sb[sp];
        if (ix->left[i] < 0) { seg_push(out, t0, t1); continue; }
        i64 li = ix->left[i], ri = ix->right[i];
        double la, lb, ra, rb;
        int hl = node_slab(r, ix, li, &la, &lb);
        if (hl) { la = la > tmin ? la : tmin; lb = lb < tmax ? lb : tmax; if (lb <= la) hl = 0; }
        int hr = node_slab(r, ix, ri, &ra, &rb);
        if (hr) { ra = ra > tmin ? ra : tmin; rb = rb < tmax ? rb : tmax; if (rb <= ra) hr = 0; }
        if (hl && hr) {
            if (la <= ra) {
                stk[sp] = ri; sa[sp] = ra; sb[sp] = rb; sp++;
                stk[sp] = li; sa[sp] = la; sb[sp] = lb; sp++;
            } else {
                stk[sp] = li; sa[sp] = la; sb[sp] = lb; sp++;
                stk[sp] = ri; sa[sp] = ra; sb[sp] = rb; sp++;
            }
        } else if (hl) { stk[sp] = li; sa[sp] = la; sb[sp] = lb; sp++; }
        else if (hr) { stk[sp] = ri; sa[sp] = ra; sb[sp] = rb; sp++; }
    }
}

/* render.py:507-562 */
static void kd_leaves(const RaySt* r, const Index* ix, double tmin, double tmax, SegBuf* out,
                      i64* stk) {
    i64 sp = 1;
    stk[0] = ix->root;
    while (sp > 0) {
        i64 i = stk[--sp];
        double a, b;
        if (!node_slab(r, ix, i, &a, &b)) continue;
        a = a > tmin ? a : tmin;
        b = b < tmax ? b : tmax;
        if (b <= a) continue;
        int ax = ix->axis[i];
        if (ax < 0) { seg_push(out, a, b); continue; }
        int front_left;
        double pl = (double)ix->plane[i];
        if ((r->zx && ax == 0) || (r->zy && ax == 1) || (r->zz && ax == 2))
            front_left = ax == 0 ? r->ox < pl : (ax == 1 ? r->oy < pl : r->oz < pl);
        else
            front_left = ax == 0 ? r->ix > 0.0 : (ax == 1 ? r->iy > 0.0 : r->iz > 0.0);
        i64 nr = front_left ? ix->left[i] : ix->right[i];
        i64 fr = front_left ? ix->right[i] : ix->left[i];
        if (fr >= 0) stk[sp++] = fr;
        if (nr >= 0) stk[sp++] = nr;
    }
}

/* Per-ray interval list exactly as _Traverser.run returns it (sorted, merged).
 * Returns the number of intervals in seg->t[0:2n]. */
static i64 traverse_ray(const Index* ix, const RaySt* r, SegBuf* seg, SegBuf* tmp, i64* stk,
                        double* sa, double* sb) {
    seg->n = 0;
    double tmin, tmax;
    if (!slab(r, 0.0, 0.0, 0.0, (double)ix->nx, (double)ix->ny, (double)ix->nz, &tmin, &tmax)) return 0;
    switch (ix->kind) {
        case 0:  /* render.py:290-302 */
            seg_push(seg, tmin, tmax);
            return 1;
        case 1:  /* render.py:381-401 */
            dda_runs(r, ix, tmin, tmax, seg);
            return sort_merge(seg->t, seg->n);
        case 2:
            if (ix->root < 0) return 0;
            bvh_leaves(r, ix, tmin, tmax, seg, stk, sa, sb);
            return sort_merge(seg->t, seg->n);
        case 3:  /* render.py:565-590 */
            if (ix->root < 0) return 0;
            kd_leaves(r, ix, tmin, tmax, seg, stk);
            return sort_merge(seg->t, seg->n);
        default: {  /* render.py:593-630 */
            if (ix->root < 0) return 0;
            tmp->n = 0;
            kd_leaves(r, ix, tmin, tmax, tmp, stk);
            i64 nleaf = sort_merge(tmp->t, tmp->n);
            for (i64 s = 0; s < nleaf; ++s) dda_runs(r, ix, tmp->t[2 * s], tmp->t[2 * s + 1], seg);
            return sort_merge(seg->t, seg->n);
        }
    }
}

/* render.py:633-765 for one ray. */
static void integrate_ray(const RaySt* r, const double* seg, i64 m, const void* field, int is_f32,
                          const float* u8tab, i64 nx, i64 ny, i64 nz, const float* lut,
                          const double* corr, double dt, int nearest, double* rgba, i64* samples) {
    rgba[0] = rgba[1] = rgba[2] = rgba[3] = 0.0;
    *samples = 0;
    if (m == 0) return;
    double entry, ex;
    if (!slab(r, 0.0, 0.0, 0.0, (double)nx, (double)ny, (double)nz, &entry, &ex)) return;
    double accr = 0.0, accg = 0.0, accb = 0.0, acca = 0.0;
    i64 taken = 0;
    for (i64 s = 0; s < m; ++s) {
        double t0 = seg[2 * s], t1 = seg[2 * s + 1];
        i64 k = (i64)ceil((t0 - entry) / dt);
        if (k < 0) k = 0;
        while (k > 0 && entry + (double)(k - 1) * dt >= t0) k--;
        while (entry + (double)k * dt < t0) k++;
        double t = entry + (double)k * dt;
        while (t < t1) {
            double px = r->ox + t * r->dx, py = r->oy + t * r->dy, pz = r->oz + t * r->dz;
            double value;
            if (nearest) {
                i64 xi = (i64)floor(px), yi = (i64)floor(py), zi = (i64)floor(pz);
                xi = xi < 0 ? 0 : (xi > nx - 1 ? nx - 1 : xi);
                yi = yi < 0 ? 0 : (yi > ny - 1 ? ny - 1 : yi);
                zi = zi < 0 ? 0 : (zi > nz - 1 ? nz - 1 : zi);
                value = (double)field_value(field, is_f32, IDX3(xi, yi, zi, ny, nz), u8tab);
            } else {
                double qx = px - 0.5, qy = py - 0.5, qz = pz - 0.5;
                i64 x0 = (i64)floor(qx), y0 = (i64)floor(qy), z0 = (i64)floor(qz);
                double fx = qx - (double)x0, fy = qy - (double)y0, fz = qz - (double)z0;
                i64 x1 = x0 + 1, y1 = y0 + 1, z1 = z0 + 1;
                x0 = x0 < 0 ? 0 : (x0 > nx - 1 ? nx - 1 : x0);
                y0 = y0 < 0 ? 0 : (y0 > ny - 1 ? ny - 1 : y0);
                z0 = z0 < 0 ? 0 : (z0 > nz - 1 ? nz - 1 : z0);
                x1 = x1 < 0 ? 0 : (x1 > nx - 1 ? nx - 1 : x1);
                y1 = y1 < 0 ? 0 : (y1 > ny - 1 ? ny - 1 : y1);
                z1 = z1 < 0 ? 0 : (z1 > nz - 1 ? nz - 1 : z1);
                float c000 = field_value(field, is_f32, IDX3(x0, y0, z0, ny, nz), u8tab);
                float c100 = field_value(field, is_f32, IDX3(x1, y0, z0, ny, nz), u8tab);
                float c010 = field_value(field, is_f32, IDX3(x0, y1, z0, ny, nz), u8tab);
                float c110 = field_value(field, is_f32, IDX3(x1, y1, z0, ny, nz), u8tab);
                float c001 = field_value(field, is_f32, IDX3(x0, y0, z1, ny, nz), u8tab);
                float c101 = field_value(field, is_f32, IDX3(x1, y0, z1, ny, nz), u8tab);
                float c011 = field_value(field, is_f32, IDX3(x0, y1, z1, ny, nz), u8tab);
                float c111 = field_value(field, is_f32, IDX3(x1, y1, z1, ny, nz), u8tab);
                /* numba types f32 - f32 as f32, then promotes (render.py:738-741) */
                float d00 = c100 - c000, d10 = c110 - c010, d01 = c101 - c001, d11 = c111 - c011;
                double c00 = (double)c000 + (double)d00 * fx;
                double c10 = (double)c010 + (double)d10 * fx;
                double c01 = (double)c001 + (double)d01 * fx;
                double c11 = (double)c011 + (double)d11 * fx;
                double c0 = c00 + (c10 - c00) * fy;
                double c1 = c01 + (c11 - c01) * fy;
                value = c0 + (c1 - c0) * fz;
            }
            double bd = floor(value * 255.0 + 0.5);
            int bin = bd < 0.0 ? 0 : (bd > 255.0 ? 255 : (int)bd);
            float alpha = lut[4 * bin + 3];
            if (alpha > 0.0f) {
                double weight = (1.0 - acca) * corr[bin];
                accr += weight * (double)lut[4 * bin + 0];
                accg += weight * (double)lut[4 * bin + 1];
                accb += weight * (double)lut[4 * bin + 2];
                acca += weight;
            }
            taken++;
            k++;
            t = entry + (double)k * dt;
        }
    }
    rgba[0] = accr; rgba[1] = accg; rgba[2] = accb; rgba[3] = acca;
    *samples = taken;
}

/* 1 - (1 - alpha)**dt with libm pow, as numba's ** (render.py:752). */
void or_corr_table(const float* lut, double dt, double* corr) {
    for (int b = 0; b < 256; ++b) corr[b] = 1.0 - pow(1.0 - (double)lut[4 * b + 3], dt);
}

/* Camera.ray_origins (render.py:134-149) for pixel (i, j): (eye + ys*up) + xs*right. */
static void pixel_origin(const double* cam, i64 w, i64 h, i64 i, i64 j, double* o) {
    const double *eye = cam, *up = cam + 3, *right = cam + 6;
    double scale = cam[9];
    double xs = (((double)i + 0.5) - (double)w / 2.0) * scale;
    double ys = (((double)h / 2.0 - (double)j) - 0.5) * scale;
    for (int a = 0; a < 3; ++a) o[a] = (eye[a] + ys * up[a]) + xs * right[a];
}

/* render_frame (render.py:869-911) over image rows [row0, row1).
 * cam = eye[3], up[3], right[3], scale (host-normalised exactly as ray_origins does).
 * rgba: (row1-row0)*w*4 float64, samples: (row1-row0)*w int64.  Rays are independent, so
 * the pthread split (dynamic chunks of 256 rays) does not change any result. */
typedef struct {
    const Index* ix;
    const void* field; int is_f32; const float* lut; const double* corr; const float* tab;
    const double* cam; const double* dir;
    i64 w, h, row0, nrays, stack_cap;
    double dt; int nearest;
    double* rgba; i64* samples;
    atomic_llong next;
} RenderJob;

static void* render_worker(void* arg) {
    RenderJob* jb = (RenderJob*)arg;
    SegBuf seg = {0, 0, 0}, tmp = {0, 0, 0};
    i64* stk = (i64*)malloc(sizeof(i64) * (size_t)(jb->stack_cap + 4));
    double* sa = (double*)malloc(sizeof(double) * (size_t)(jb->stack_cap + 4));
    double* sb = (double*)malloc(sizeof(double) * (size_t)(jb->stack_cap + 4));
    const Index* ix = jb->ix;
    for (;;) {
        i64 q0 = atomic_fetch_add(&jb->next, 256);
        if (q0 >= jb->nrays) break;
        i64 q1 = q0 + 256 < jb->nrays ? q0 + 256 : jb->nrays;
        for (i64 q = q0; q < q1; ++q) {
            i64 j = jb->row0 + q / jb->w, i = q % jb->w;
            double o[3];
            pixel_origin(jb->cam, jb->w, jb->h, i, j, o);
            RaySt r;
            ray_setup(&r, o, jb->dir);
            i64 m = traverse_ray(ix, &r, &seg, &tmp, stk, sa, sb);
            integrate_ray(&r, seg.t, m, jb->field, jb->is_f32, jb->tab, ix->nx, ix->ny, ix->nz,
                          jb->lut, jb->corr, jb->dt, jb->nearest, jb->rgba + 4 * q, jb->samples + q);
        }
    }
    free(seg.t); free(tmp.t); free(stk); free(sa); free(sb);
    return NULL;
}

void or_render(int kind, const void* field, int is_f32, i64 nx, i64 ny, i64 nz, const float* lut,
               const uint8_t* occ, i64 ncx, i64 ncy, i64 ncz, i64 cs, const int32_t* lo,
               const int32_t* hi, const int32_t* left, const int32_t* right, const int8_t* axis,
               const int32_t* plane, i64 root, i64 stack_cap, const double* cam, const double* dir,
               i64 w, i64 h, i64 row0, i64 row1, double dt, int nearest, double* rgba, i64* samples,
               int nthreads) {
    Index ix = {kind, nx, ny, nz, occ, ncx, ncy, ncz, (double)cs, lo, hi, left, right, plane, axis, root};
    float tab[256];
    or_u8_field_table(tab);
    double corr[256];
    or_corr_table(lut, dt, corr);
    RenderJob jb;
    jb.ix = &ix; jb.field = field; jb.is_f32 = is_f32; jb.lut = lut; jb.corr = corr; jb.tab = tab;
    jb.cam = cam; jb.dir = dir; jb.w = w; jb.h = h; jb.row0 = row0; jb.nrays = (row1 - row0) * w;
    jb.stack_cap = stack_cap; jb.dt = dt; jb.nearest = nearest; jb.rgba = rgba; jb.samples = samples;
    atomic_init(&jb.next, 0);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, render_worker, &jb);
    render_worker(&jb);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* Single-ray traversal (render.py:928-961): writes up to cap intervals, returns count. */
i64 or_traverse(int kind, i64 nx, i64 ny, i64 nz, const uint8_t* occ, i64 ncx, i64 ncy, i64 ncz,
                i64 cs, const int32_t* lo, const int32_t* hi, const int32_t* left,
                const int32_t* right, const int8_t* axis, const int32_t* plane, i64 root,
                i64 stack_cap, const double* origin, const double* dir, double* out, i64 cap) {
    Index ix = {kind, nx, ny, nz, occ, ncx, ncy, ncz, (double)cs, lo, hi, left, right, plane, axis, root};
    SegBuf seg = {0, 0, 0}, tmp = {0, 0, 0};
    i64* stk = (i64*)malloc(sizeof(i64) * (size_t)(stack_cap + 4));
    double* sa = (double*)malloc(sizeof(double) * (size_t)(stack_cap + 4));
    double* sb = (double*)malloc(sizeof(double) * (size_t)(stack_cap + 4));
    RaySt r;
    ray_setup(&r, origin, dir);
    i64 m = traverse_ray(&ix, &r, &seg, &tmp, stk, sa, sb);
    for (i64 s = 0; s < m && s < cap; ++s) { out[2 * s] = seg.t[2 * s]; out[2 * s + 1] = seg.t[2 * s + 1]; }
    free(seg.t); free(tmp.t); free(stk); free(sa); free(sb);
    return m;
}

/* Single-ray integration (render.py:964-1015). */
void or_integrate(const double* origin, const double* dir, const double* seg, i64 m,
                  const void* field, int is_f32, i64 nx, i64 ny, i64 nz, const float* lut,
                  double dt, int nearest, double* rgba, i64* samples) {
    float tab[256];
    or_u8_field_table(tab);
    double corr[256];
    or_corr_table(lut, dt, corr);
    RaySt r;
    ray_setup(&r, origin, dir);
    integrate_ray(&r, seg, m, field, is_f32, tab, nx, ny, nz, lut, corr, dt, nearest, rgba, samples);
}

/* ------------------------------------------------------------------------------------ */
/* Multi-channel integration (BASELINE configs[4]; no reference equivalent -- "parity       */
/* unpinned" except when all channels but one have zero alpha, where it IS _k_integrate,    */
/* render.py:633-765).  Channels are composited in channel order at each lattice sample     */
/* with the reference's update.  u8 channels only.                                          */
/* ------------------------------------------------------------------------------------ */
static double trilinear_u8(const uint8_t* f, const float* tab, i64 nx, i64 ny, i64 nz, double px,
                           double py, double pz) {
    double qx = px - 0.5, qy = py - 0.5, qz = pz - 0.5;
    i64 x0 = (i64)floor(qx), y0 = (i64)floor(qy), z0 = (i64)floor(qz);
    double fx = qx - (double)x0, fy = qy - (double)y0, fz = qz - (double)z0;
    i64 x1 = x0 + 1, y1 = y0 + 1, z1 = z0 + 1;
    x0 = x0 < 0 ? 0 : (x0 > nx - 1 ? nx - 1 : x0);
    y0 = y0 < 0 ? 0 : (y0 > ny - 1 ? ny - 1 : y0);
    z0 = z0 < 0 ? 0 : (z0 > nz - 1 ? nz - 1 : z0);
    x1 = x1 < 0 ? 0 : (x1 > nx - 1 ? nx - 1 : x1);
    y1 = y1 < 0 ? 0 : (y1 > ny - 1 ? ny - 1 : y1);
    z1 = z1 < 0 ? 0 : (z1 > nz - 1 ? nz - 1 : z1);
    float c000 = tab[f[IDX3(x0, y0, z0, ny, nz)]], c100 = tab[f[IDX3(x1, y0, z0, ny, nz)]];
    float c010 = tab[f[IDX3(x0, y1, z0, ny, nz)]], c110 = tab[f[IDX3(x1, y1, z0, ny, nz)]];
    float c001 = tab[f[IDX3(x0, y0, z1, ny, nz)]], c101 = tab[f[IDX3(x1, y0, z1, ny, nz)]];
    float c011 = tab[f[IDX3(x0, y1, z1, ny, nz)]], c111 = tab[f[IDX3(x1, y1, z1, ny, nz)]];
    float d00 = c100 - c000, d10 = c110 - c010, d01 = c101 - c001, d11 = c111 - c011;
    double c00 = (double)c000 + (double)d00 * fx;
    double c10 = (double)c010 + (double)d10 * fx;
    double c01 = (double)c001 + (double)d01 * fx;
    double c11 = (double)c011 + (double)d11 * fx;
    double c0 = c00 + (c10 - c00) * fy;
    double c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

static void integrate_ray_multi(const RaySt* r, const double* seg, i64 m, const uint8_t** fields,
                                int nch, const float* u8tab, i64 nx, i64 ny, i64 nz,
                                const float** luts, const double** corrs, double dt,
                                double* rgba, i64* samples) {
    rgba[0] = rgba[1] = rgba[2] = rgba[3] = 0.0;
    *samples = 0;
    if (m == 0) return;
    double entry, ex;
    if (!slab(r, 0.0, 0.0, 0.0, (double)nx, (double)ny, (double)nz, &entry, &ex)) return;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    i64 taken = 0;
    for (i64 s = 0; s < m; ++s) {
        double t0 = seg[2 * s], t1 = seg[2 * s + 1];
        i64 k = (i64)ceil((t0 - entry) / dt);
        if (k < 0) k = 0;
        while (k > 0 && entry + (double)(k - 1) * dt >= t0) k--;
        while (entry + (double)k * dt < t0) k++;
        double t = entry + (double)k * dt;
        while (t < t1) {
            double px = r->ox + t * r->dx, py = r->oy + t * r->dy, pz = r->oz + t * r->dz;
            for (int c = 0; c < nch; ++c) {
                double value = trilinear_u8(fields[c], u8tab, nx, ny, nz, px, py, pz);
                double bd = floor(value * 255.0 + 0.5);
                int bin = bd < 0.0 ? 0 : (bd > 255.0 ? 255 : (int)bd);
                const float* lut = luts[c];
                if (lut[4 * bin + 3] > 0.0f) {
                    double w = (1.0 - acc[3]) * corrs[c][bin];
                    acc[0] += w * (double)lut[4 * bin + 0];
                    acc[1] += w * (double)lut[4 * bin + 1];
                    acc[2] += w * (double)lut[4 * bin + 2];
                    acc[3] += w;
                }
            }
            taken++;
            k++;
            t = entry + (double)k * dt;
        }
    }
    rgba[0] = acc[0]; rgba[1] = acc[1]; rgba[2] = acc[2]; rgba[3] = acc[3];
    *samples = taken;
}

/* Multi-channel frame (single thread per call; small test frames). */
typedef struct {
    const Index* ix; const uint8_t** fields; int nch; const float* tab; const float** luts;
    const double** corrs; const double* cam; const double* dir; i64 w, h, row0, nrays, stack_cap;
    double dt; double* rgba; i64* samples; atomic_llong next;
} MultiJob;

static void* render_multi_worker(void* arg) {
    MultiJob* jb = (MultiJob*)arg;
    SegBuf seg = {0, 0, 0}, tmp = {0, 0, 0};
    i64* stk = (i64*)malloc(sizeof(i64) * (size_t)(jb->stack_cap + 4));
    double* sa = (double*)malloc(sizeof(double) * (size_t)(jb->stack_cap + 4));
    double* sb = (double*)malloc(sizeof(double) * (size_t)(jb->stack_cap + 4));
    const Index* ix = jb->ix;
    for (;;) {
        i64 q0 = atomic_fetch_add(&jb->next, 256);
        if (q0 >= jb->nrays) break;
        i64 q1 = q0 + 256 < jb->nrays ? q0 + 256 : jb->nrays;
        for (i64 q = q0; q < q1; ++q) {
            double o[3];
            pixel_origin(jb->cam, jb->w, jb->h, q % jb->w, jb->row0 + q / jb->w, o);
            RaySt r;
            ray_setup(&r, o, jb->dir);
            i64 m = traverse_ray(ix, &r, &seg, &tmp, stk, sa, sb);
            integrate_ray_multi(&r, seg.t, m, jb->fields, jb->nch, jb->tab, ix->nx, ix->ny, ix->nz,
                                jb->luts, jb->corrs, jb->dt, jb->rgba + 4 * q, jb->samples + q);
        }
    }
    free(seg.t); free(tmp.t); free(stk); free(sa); free(sb);
    return NULL;
}

/* Rows [row0, row1) of a multi-channel frame, rays dealt to nthreads host threads in chunks
 * of 256 (the split never changes a ray's result). */
void or_render_multi_rows(int kind, const uint8_t** fields, int nch, i64 nx, i64 ny, i64 nz,
                          const float** luts, const uint8_t* occ, i64 ncx, i64 ncy, i64 ncz,
                          i64 cs, const int32_t* lo, const int32_t* hi, const int32_t* left,
                          const int32_t* right, const int8_t* axis, const int32_t* plane,
                          i64 root, i64 stack_cap, const double* cam, const double* dir, i64 w,
                          i64 h, i64 row0, i64 row1, double dt, double* rgba, i64* samples,
                          int nthreads) {
    Index ix = {kind, nx, ny, nz, occ, ncx, ncy, ncz, (double)cs, lo, hi, left, right, plane, axis, root};
    float tab[256];
    or_u8_field_table(tab);
    double corr_store[4][256];
    const double* corrs[4];
    for (int c = 0; c < nch; ++c) {
        or_corr_table(luts[c], dt, corr_store[c]);
        corrs[c] = corr_store[c];
    }
    MultiJob jb;
    jb.ix = &ix; jb.fields = fields; jb.nch = nch; jb.tab = tab; jb.luts = luts; jb.corrs = corrs;
    jb.cam = cam; jb.dir = dir; jb.w = w; jb.h = h; jb.row0 = row0; jb.nrays = (row1 - row0) * w;
    jb.stack_cap = stack_cap; jb.dt = dt; jb.rgba = rgba; jb.samples = samples;
    atomic_init(&jb.next, 0);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, render_multi_worker, &jb);
    render_multi_worker(&jb);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

void or_render_multi(int kind, const uint8_t** fields, int nch, i64 nx, i64 ny, i64 nz,
                     const float** luts, const uint8_t* occ, i64 ncx, i64 ncy, i64 ncz, i64 cs,
                     const int32_t* lo, const int32_t* hi, const int32_t* left,
                     const int32_t* right, const int8_t* axis, const int32_t* plane, i64 root,
                     i64 stack_cap, const double* cam, const double* dir, i64 w, i64 h,
                     double dt, double* rgba, i64* samples) {
    or_render_multi_rows(kind, fields, nch, nx, ny, nz, luts, occ, ncx, ncy, ncz, cs, lo, hi, left,
                         right, axis, plane, root, stack_cap, cam, dir, w, h, 0, h, dt, rgba,
                         samples, 1);
}
